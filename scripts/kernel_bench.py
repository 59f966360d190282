"""BASELINE.json configs[5] kernel microbenchmark (n = 4096, 33.6 M DOF, seed 4, log-uniform
viscosity 1e4..1e13 per cell, state v = 0, pi = 0 (reading G24)): times the fused residual +
Jacobian assembly, one SpMV, one Chebyshev(3) V-cycle and one 30-vector FGMRES cycle
(rtol = 0, exactly 30 iterations) separately, median of `--reps` after 3 warm-ups, CUDA events;
reports algorithmic GB/s against the measured copy bandwidth.  One JSON line."""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2204_10822_b200 import workloads as wl
from paper_2204_10822_b200.seaice import SeaIce

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
cfg = wl.CONFIGS[a.config]
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
inp = wl.step_inputs(cfg, 0)
ctx = SeaIce(cfg.n, krylov_rtol=0.0, krylov_maxit=30, restart=30)
ctx.set_inputs(inp)
N, Nn, Nc = ctx.N, (cfg.n + 1) ** 2, cfg.n * cfg.n
v = torch.zeros(N, dtype=torch.float64, device="cuda")


def timed(fn, reps=a.reps):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


out = {"workload": cfg.name, "n": cfg.n, "dof": N, "peak_gbs": peak}
ms = timed(lambda: ctx.assemble_jacobian(v, None, want_csr=False))
b = 216.0 * Nn + 112.0 * Nc  # symmetric stencil (19 x 8 B) + v, v_o, F, R per node; pi, P, rho h per cell
ctx.profile(True)
for _ in range(3):
    ctx.assemble_jacobian(v, None, want_csr=False)
pa = ctx.profile_read()["assemble"]
ctx.profile(False)
kms = pa["ms"] / max(pa["launches"], 1)
out["assembly"] = {"ms": ms, "kernel_ms": kms, "alg_bytes": b, "gbs": b / kms / 1e6, "frac": b / kms / 1e6 / peak,
                   "api_gbs": b / ms / 1e6,
                   "note": "kernel time from CUDA events around the launch; ms includes the API's reduction + sync"}
x = torch.randn(N, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
ms = timed(lambda: ctx.spmv(x))
b = 184.0 * Nn  # symmetric stencil (152 B) + x, y per node
out["spmv"] = {"ms": ms, "alg_bytes": b, "gbs": b / ms / 1e6, "frac": b / ms / 1e6 / peak}
# NEXT-4: matrix-free apply of the same operator (element algebra recomputed per call)
yb = torch.empty_like(x)
ms = timed(lambda: ctx.jv_matfree(v, x))
b = 64.0 * Nn + 112.0 * Nc
out["jv_matfree"] = {"ms": ms, "alg_bytes": b, "gbs": b / ms / 1e6, "frac": b / ms / 1e6 / peak,
                     "vs_spmv": ms / out["spmv"]["ms"],
                     "note": "fp64-bound: per-cell element algebra recomputed each apply (ms incl. the binding's output allocation)"}
nl, oc = ctx.amg_setup()
out["amg"] = {"levels": nl, "op_complexity": oc, "setup_ms": timed(lambda: ctx.amg_setup(), reps=3)}
ms = timed(lambda: ctx.precond_apply(x))
ctx.profile(True)
ctx.precond_apply(x)
p = ctx.profile_read()
ctx.profile(False)
vb = sum(d["bytes"] for d in p.values())
out["vcycle"] = {"ms": ms, "alg_bytes": vb, "gbs": vb / ms / 1e6, "frac": vb / ms / 1e6 / peak,
                 "note": "graph replay incl. in/out copies; bytes from the per-kernel formulas"}
R, _ = ctx.residual(v)
ctx.assemble_jacobian(v, None, want_csr=False)
ctx.amg_setup()
res = {}


def cyc():
    xx, st, rc = ctx.fgmres(R)
    res.update(st)


ms = timed(cyc, reps=3)
out["fgmres_cycle"] = {"ms": ms, "iters": res.get("iters"), "ms_per_iter": ms / max(res.get("iters", 1), 1),
                       "dof_iters_per_s": N * res.get("iters", 0) / (ms / 1e3)}
print(json.dumps(out))
