"""NEXT-1 / NEXT-2 rows: the paper's Problem I on the GPU path.

* sv Newton to a 1e4 residual reduction at dx = 4, 2, 1, 0.5, 0.25 km; the paper
  reports 30 / 37 / 45 iterations at 1 / 0.5 / 0.25 km (context, other codes).
* standard Newton (eq:standardNewton) and Picard at the same settings: the paper reports that
  standard Newton "makes little progress within 200 iterations" at 1 km.
Prints one JSON line per run."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2204_10822_b200 import workloads as wl
from paper_2204_10822_b200.seaice import SeaIce

ap = argparse.ArgumentParser()
ap.add_argument("--sizes", default="128,256,512,1024,2048")
ap.add_argument("--kinds", default="sv")
ap.add_argument("--maxit", type=int, default=200)
ap.add_argument("--params", default="{}")
a = ap.parse_args()
PAPER = {512: 30, 1024: 37, 2048: 45}
for kind in a.kinds.split(","):
    for n in [int(x) for x in a.sizes.split(",")]:
        inp = wl.problem1_inputs(n)
        ctx = SeaIce(n, f_c=0.0, newton_rtol=1e-4, newton_maxit=a.maxit, jacobian=kind, **json.loads(a.params))
        torch.cuda.synchronize()
        t0 = time.time()
        v, st = ctx.solve_step(inp.dt, inp.t_new, inp.h, inp.A, inp.v_prev, inp.v_air, inp.v_ocean)
        torch.cuda.synchronize()
        rec = {"problem": "I", "kind": kind, "n": n, "dx_km": 512.0 / n, "newton": st["newton_iters"],
               "converged": st["converged"], "relres_final": st["res_norm_final"] / st["res_norm0"],
               "krylov_total": st["krylov_iters_total"], "amg_setups": st["amg_setups"], "seconds": round(time.time() - t0, 2),
               "paper_sv_newton": PAPER.get(n) if kind == "sv" else None,
               "vmax": float(v.abs().max())}
        print(json.dumps(rec), flush=True)
        ctx.close()
        del ctx
        torch.cuda.empty_cache()
