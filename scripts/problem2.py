"""NEXT-3 row: the paper's Problem II time loop (Mehlmann 2021 benchmark) on the GPU
path — per step: explicit upwind transport of A and H with v^n (seaice_transport),
then the implicit sv-Newton momentum step at t_{n+1} (seaice_solve_step), with the paper's
settings: f_c = 0, Delta_min = 2e-9, dt = 0.5 h, Newton to a 1e4 residual reduction
(P:724-726).  Context (other codes/hardware, P:913-933 Table `meaniter`, P:1043-1045 Fig. `amg`):
mean Newton iterations 6.66 / 11.32 / 15.91 / 20.20 and mean Krylov iterations per solve
14 / 17 / 22 / 30 at 4 / 2 / 1 / 0.5 km over 8 days (384 steps).
Prints one JSON line per run (plus per-step lines with --per-step)."""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2204_10822_b200 import workloads as wl
from paper_2204_10822_b200.seaice import SeaIce

ap = argparse.ArgumentParser()
ap.add_argument("--runs", default="128:384,256:384,512:384,1024:48", help="n:steps,...")
ap.add_argument("--per-step", action="store_true")
ap.add_argument("--params", default="{}")
a = ap.parse_args()
PAPER_NEWTON = {128: 6.66, 256: 11.32, 512: 15.91, 1024: 20.20}
PAPER_KRYLOV = {128: 14, 256: 17, 512: 22, 1024: 30}
dt = 1800.0
for run in a.runs.split(","):
    n, steps = (int(x) for x in run.split(":"))
    ctx = SeaIce(n, f_c=0.0, newton_rtol=1e-4, **json.loads(a.params))
    h0, A0, v0 = wl.problem2_initial(n)
    vo = torch.as_tensor(wl.ocean_nodal(n), device="cuda")
    h, A, v = (torch.as_tensor(x, device="cuda") for x in (h0, A0, v0))
    newton, krylov, secs, tsec, conv, cfls, subs = [], [], [], [], 0, [], []
    ctx_capped = 0
    for k in range(steps):
        t_new = (k + 1) * dt
        va = torch.as_tensor(wl.problem2_wind_nodal(n, t_new), device="cuda")
        torch.cuda.synchronize()
        t0 = time.time()
        A, h, cfl, msub = ctx.transport(dt, v, A, h, info=True)
        cfls.append(cfl)
        subs.append(msub)
        torch.cuda.synchronize()
        t1 = time.time()
        v, st = ctx.solve_step(dt, t_new, h, A, v, va, vo)
        torch.cuda.synchronize()
        t2 = time.time()
        newton.append(st["newton_iters"])
        krylov.append(st["krylov_iters_total"])
        secs.append(t2 - t1)
        tsec.append(t1 - t0)
        conv += st["converged"]
        ctx_capped += st["krylov_capped"]
        if a.per_step:
            print(json.dumps({"n": n, "step": k + 1, "day": t_new / wl.DAY, "newton": st["newton_iters"],
                              "krylov": st["krylov_iters_total"], "seconds": round(t2 - t1, 4), "cfl": cfl,
                              "A_min": float(A.min()), "h_max": float(h.max())}), flush=True)
    rec = {"problem": "II", "n": n, "dx_km": 512.0 / n, "dof": ctx.N, "steps": steps, "days": steps * dt / wl.DAY,
           "converged_steps": conv, "newton_mean": statistics.mean(newton), "newton_max": max(newton),
           "krylov_per_solve": sum(krylov) / max(sum(newton), 1), "s_per_step": statistics.mean(secs),
           "transport_us_per_step": 1e6 * statistics.median(tsec), "cfl_max": max(cfls),
           "transport_substeps_max": max(subs), "krylov_capped": ctx_capped,
           "paper_newton_mean_8d": PAPER_NEWTON.get(n), "paper_krylov_per_solve_8d": PAPER_KRYLOV.get(n),
           "A_min": float(A.min()), "A_max": float(A.max()), "h_min": float(h.min()), "h_max": float(h.max())}
    print(json.dumps(rec), flush=True)
    ctx.close()
    del ctx
    torch.cuda.empty_cache()
