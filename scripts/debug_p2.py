"""Development aid: find Problem II steps whose Newton loop does not converge and replay them
with per-iteration statistics (and with alternative parameter sets)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2204_10822_b200 import workloads as wl
from paper_2204_10822_b200.seaice import SeaIce

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--steps", type=int, default=192)
ap.add_argument("--params", default="{}")
ap.add_argument("--alts", default='[{"krylov_forcing":0},{"nullspace_dim":3}]')
ap.add_argument("--iters", type=int, default=60)
a = ap.parse_args()
n, dt = a.n, 1800.0
base = dict(f_c=0.0, newton_rtol=1e-4, **json.loads(a.params))
ctx = SeaIce(n, **base)
h0, A0, v0 = wl.problem2_initial(n)
vo = torch.as_tensor(wl.ocean_nodal(n), device="cuda")
h, A, v = (torch.as_tensor(x, device="cuda") for x in (h0, A0, v0))


def replay(params, A, h, v, va, t_new, iters):
    c = SeaIce(n, **params)
    c.set_step(dt, t_new, h, A, v, va, vo)
    vv = v.clone()
    rows = []
    for l in range(iters):
        d = c.newton_step(vv)
        if d["converged_on_entry"]:
            rows.append({"l": l, "converged": True, "res": d["res_norm"] / d["res_norm0"]})
            break
        rows.append({"l": l, "res": d["res_norm"] / d["res_norm0"], "alpha": d["alpha"], "halv": d["halvings"],
                     "stag": d["ls_stagnated"], "kry": d["krylov"]["iters"], "krel": d["krylov"]["relres_true"],
                     "dphi": d["dphi"]})
    c.close()
    return rows


for k in range(a.steps):
    t_new = (k + 1) * dt
    va = torch.as_tensor(wl.problem2_wind_nodal(n, t_new), device="cuda")
    A, h, cfl, msub = ctx.transport(dt, v, A, h, info=True)
    v_before = v.clone()
    v, st = ctx.solve_step(dt, t_new, h, A, v, va, vo)
    if not st["converged"] or st["newton_iters"] >= 60:
        print(json.dumps({"step": k + 1, "newton": st["newton_iters"], "converged": st["converged"], "cfl": cfl}),
              flush=True)
        for p in [base] + [dict(base, **x) for x in json.loads(a.alts)]:
            rows = replay(p, A, h, v_before, va, t_new, a.iters)
            print(json.dumps({"params": p, "n_iters": len(rows), "last": rows[-1]}), flush=True)
            for r in rows[:a.iters]:
                print("   ", json.dumps(r), flush=True)
        break
