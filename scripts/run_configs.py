"""Run BASELINE.json configs 1-4 end to end on the GPU (every implicit step of each config)
and record per-step Newton/FGMRES counts and times.  Writes JSON lines to stdout.  (Parity with
the oracle is the job of tests/: tests/test_gpu_goldens.py compares configs 2 and 3 with stored
oracle results; this script does not run the oracle.)"""
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
ap.add_argument("--params", default="{}")
a = ap.parse_args()

for cid in [int(x) for x in a.configs.split(",")]:
    cfg = wl.CONFIGS[cid]
    ctx = SeaIce(cfg.n, **json.loads(a.params))
    hA = wl.ice_fields(cfg)
    h, A = hA
    vo = wl.ocean_nodal(cfg.n)
    v = torch.zeros(ctx.N, dtype=torch.float64, device="cuda")
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
               "t_amg_ms": round(st["t_amg"], 1), "t_krylov_ms": round(st["t_krylov"], 1),
               "krylov_capped": st["krylov_capped"], "amg_setups": st["amg_setups"]}
        print(json.dumps(rec), flush=True)
        v = vn
    ctx.close()
    del ctx
    torch.cuda.empty_cache()
