"""Run BASELINE.json configs 1-4 end to end on the GPU (every implicit step of each config)
and record per-step Newton/FGMRES counts, times and (where the oracle finishes in minutes)
parity with the CPU oracle (direct solves).  Writes JSON lines to stdout."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2204_10822_b200 import workloads as wl
from paper_2204_10822_b200.seaice import SeaIce

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="1,2,3,4")
ap.add_argument("--oracle-steps", default="1:1,2:1", help="config:steps compared with the oracle")
a = ap.parse_args()
oracle_steps = {int(k): int(v) for k, v in (x.split(":") for x in a.oracle_steps.split(",") if x)}
prm = wl.PhysParams()

for cid in [int(x) for x in a.configs.split(",")]:
    cfg = wl.CONFIGS[cid]
    ctx = SeaIce(cfg.n)
    hA = wl.ice_fields(cfg)
    h, A = hA
    vo = wl.ocean_nodal(cfg.n)
    v = torch.zeros(ctx.N, dtype=torch.float64, device="cuda")
    v_or = None
    zeta = None
    for s in range(cfg.steps):
        t_new = (s + 1) * cfg.dt
        va = wl.wind_nodal(cfg.n, t_new, cfg.moving)
        torch.cuda.synchronize()
        t0 = time.time()
        vn, st = ctx.solve_step(cfg.dt, t_new, h, A, v, va, vo)
        torch.cuda.synchronize()
        wall = time.time() - t0
        rec = {"config": cid, "n": cfg.n, "dof": ctx.N, "step": s + 1, "newton": st["newton_iters"],
               "krylov_total": st["krylov_iters_total"], "converged": st["converged"], "seconds": round(wall, 3),
               "relres_final": st["res_norm_final"] / max(st["res_norm0"], 1e-300),
               "t_amg_ms": round(st["t_amg"], 1), "t_krylov_ms": round(st["t_krylov"], 1)}
        if s < oracle_steps.get(cid, 0):
            from oracle import newton
            inp = wl.step_inputs(cfg, s, v_prev=v_or if v_or is not None else None, h_A=hA)
            to = time.time()
            vo_, _, ho = newton.solve_step(inp, prm)
            rec.update({"oracle_newton": ho["newton_iters"], "oracle_seconds": round(time.time() - to, 1),
                        "v_rel_l2_vs_oracle": float(np.linalg.norm(vn.cpu().numpy() - vo_) / np.linalg.norm(vo_))})
            v_or = vo_
        # viscosity spread of the converged state (G25): zeta = P/(2 Delta) per cell (from pi:
        # Delta is not exported; use the residual-consistent state through the oracle formula on a sample)
        print(json.dumps(rec), flush=True)
        v = vn
    ctx.close()
    del ctx
    torch.cuda.empty_cache()
