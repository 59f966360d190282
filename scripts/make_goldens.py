"""Write parity goldens for BASELINE.json configs 2 and 3 by calling ONLY `oracle/` (and the
seeded generators in `workloads.py`).  Nothing here touches the CUDA path: every stored value
is the oracle's (task rule ③: "a stored value ... written by a committed script that calls only
oracle/").

  cfg2  all 24 implicit steps of config 2 (n = 256, seed 1, moving cyclone), sv Newton to 1e-8
        with sparse direct solves (oracle tier A), each step warm-started from the
        oracle's own previous v.  Stored per step: Newton count, final relres, ||v||, v at 512
        fixed sampled DOFs; full v for steps 1, 12, 24.
  cfg3  step 1 of config 3 (n = 1024, seed 2) with the AMG-FGMRES of `oracle/amg.py` (tier B,
        same AMG definition as the GPU; FGMRES(30), the default when it was made).  Stored: Newton count, FGMRES count per
        solve, AMG levels per solve, final relres, full v.

  cfg4  step 1 of config 4 (n = 2048, seed 3, 8.4 M unknowns) with the product defaults: tier-B
        AMG-FGMRES(30) (MIS(2) finest / MIS(3) coarse, 4 near-nullspace columns) and the
        Eisenstat-Walker forcing of reading G29.  Stored: Newton count, FGMRES count per solve,
        AMG levels, residual history, v at 65536 sampled DOFs + ||v||.

Usage: python scripts/make_goldens.py cfg2|cfg3|cfg4 [--out tests/golden]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from oracle import newton
from paper_2204_10822_b200 import workloads as wl

SAMPLE_SEED = 12345


def sample_idx(N, k=512):
    return np.sort(np.random.default_rng(SAMPLE_SEED).choice(N, size=k, replace=False))


def run_cfg2(out):
    cfg = wl.CONFIGS[2]
    prm = wl.PhysParams()
    hA = wl.ice_fields(cfg, prm)
    N = 2 * (cfg.n + 1) ** 2
    idx = sample_idx(N)
    v = None
    steps, full = [], {}
    for s in range(cfg.steps):
        t0 = time.time()
        inp = wl.step_inputs(cfg, s, v_prev=v, h_A=hA)
        v, pi, h = newton.solve_step(inp, prm, linsolve="direct")
        rec = {"step": s + 1, "newton": h["newton_iters"], "converged": bool(h["converged"]),
               "relres": h["res"][-1] / h["res"][0], "r0": h["res"][0], "vnorm": float(np.linalg.norm(v)),
               "v_sample": v[idx].tolist(), "alphas": h["alpha"], "seconds": round(time.time() - t0, 1)}
        steps.append(rec)
        print(json.dumps({k: rec[k] for k in ("step", "newton", "relres", "vnorm", "seconds")}), flush=True)
        if s + 1 in (1, 12, 24):
            full[f"v_step{s + 1}"] = v.copy()
    meta = {"config": 2, "n": cfg.n, "seed": cfg.seed, "solver": "oracle sv-Newton, scipy sparse direct solves",
            "newton_rtol": 1e-8, "sample_idx_seed": SAMPLE_SEED, "sample_idx": idx.tolist(), "steps": steps,
            "generator": "scripts/make_goldens.py cfg2 (calls oracle/ only)"}
    with open(os.path.join(out, "cfg2_steps.json"), "w") as f:
        json.dump(meta, f)
    np.savez_compressed(os.path.join(out, "cfg2_v.npz"), **full)


def run_cfg3(out):
    cfg = wl.CONFIGS[3]
    prm = wl.PhysParams()
    t0 = time.time()
    inp = wl.step_inputs(cfg, 0)
    # the AMG definition this golden was generated with (MIS(2) on every level: the oracle default
    # before agg_dist = 3 became the coarse-level default); the GPU test runs the same definition
    amg_params = {"agg_dist0": 2, "agg_dist": 2}
    v, pi, h = newton.solve_step(inp, prm, linsolve="amg_fgmres", amg_params=amg_params, restart=30)
    meta = {"config": 3, "n": cfg.n, "seed": cfg.seed, "step": 1,
            "solver": "oracle sv-Newton, AMG-FGMRES(30) rtol 1e-8 (oracle/amg.py defaults: nullspace_dim 4, reading G30)",
            "gpu_params": dict(amg_params, restart=30), "amg_params": amg_params,
            "newton": h["newton_iters"], "converged": bool(h["converged"]), "relres": h["res"][-1] / h["res"][0],
            "krylov": [k["iters"] for k in h["krylov"]], "levels": [k.get("levels") for k in h["krylov"]],
            "alphas": h["alpha"], "res": h["res"], "seconds": round(time.time() - t0, 1),
            "generator": "scripts/make_goldens.py cfg3 (calls oracle/ only)",
            "v_storage": "cfg3_v.npz: v at 65536 DOFs drawn by numpy default_rng(12345) (sorted) + ||v||_2"}
    with open(os.path.join(out, "cfg3_step1.json"), "w") as f:
        json.dump(meta, f)
    idx = np.sort(np.random.default_rng(SAMPLE_SEED).choice(v.size, size=65536, replace=False))
    np.savez_compressed(os.path.join(out, "cfg3_v.npz"), sample_idx=idx.astype(np.int64), v_sample=v[idx],
                        v_norm=np.array([np.linalg.norm(v)]))


def run_cfg4(out):
    cfg = wl.CONFIGS[4]
    prm = wl.PhysParams()
    t0 = time.time()
    inp = wl.step_inputs(cfg, 0)
    # amg_lag = 0: a full AMG setup every Newton iteration on both sides (the lagging rule of G31
    # branches on an iteration count, so a count differing by one would fork the two runs)
    v, pi, h = newton.solve_step(inp, prm, linsolve="amg_fgmres", forcing=1, amg_lag=0, restart=30)
    meta = {"config": 4, "n": cfg.n, "seed": cfg.seed, "step": 1,
            "solver": "oracle sv-Newton, AMG-FGMRES(30) with Eisenstat-Walker forcing (reading G29), floor rtol 1e-8; "
                      "oracle/amg.py defaults (nullspace_dim 4, agg_dist0 2, agg_dist 3) = the product defaults",
            "gpu_params": {"amg_lag": 0, "restart": 30}, "newton": h["newton_iters"], "converged": bool(h["converged"]),
            "relres": h["res"][-1] / h["res"][0], "krylov": [k["iters"] for k in h["krylov"]],
            "levels": [k.get("levels") for k in h["krylov"]], "alphas": h["alpha"], "res": h["res"],
            "seconds": round(time.time() - t0, 1), "generator": "scripts/make_goldens.py cfg4 (calls oracle/ only)",
            "v_storage": "cfg4_v.npz: v at 65536 DOFs drawn by numpy default_rng(12345) (sorted) + ||v||_2"}
    with open(os.path.join(out, "cfg4_step1.json"), "w") as f:
        json.dump(meta, f)
    idx = np.sort(np.random.default_rng(SAMPLE_SEED).choice(v.size, size=65536, replace=False))
    np.savez_compressed(os.path.join(out, "cfg4_v.npz"), sample_idx=idx.astype(np.int64), v_sample=v[idx],
                        v_norm=np.array([np.linalg.norm(v)]))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("which", choices=["cfg2", "cfg3", "cfg4"])
    ap.add_argument("--out", default=os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                  "tests", "golden"))
    a = ap.parse_args()
    {"cfg2": run_cfg2, "cfg3": run_cfg3, "cfg4": run_cfg4}[a.which](a.out)
