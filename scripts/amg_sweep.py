"""AMG parameter sweep on GPU at a late sv-Newton iterate (development aid).

Runs the product Newton loop on a config to iteration --iterate, then for each parameter
set builds a fresh hierarchy for that (v, pi) and reports FGMRES iterations, setup and
solve times."""
import argparse
import itertools
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2204_10822_b200 import workloads as wl
from paper_2204_10822_b200.seaice import SeaIce

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--iterates", default="3,10")
ap.add_argument("--grid", default='{"amg_theta":[0.08]}')
a = ap.parse_args()
cfg = wl.CONFIGS[a.config]
h, A = wl.ice_fields(cfg)
va = wl.wind_nodal(cfg.n, cfg.dt, cfg.moving)
vo = wl.ocean_nodal(cfg.n)
v0 = torch.zeros(2 * (cfg.n + 1) ** 2, dtype=torch.float64, device="cuda")
its = sorted(int(x) for x in a.iterates.split(","))
base = SeaIce(cfg.n)
base.set_step(cfg.dt, cfg.dt, h, A, v0, va, vo)
v = v0.clone()
states = {}
for l in range(max(its) + 1):
    if l in its:
        states[l] = (v.clone(), base.get_pi().clone())
    d = base.newton_step(v)
    if d["converged_on_entry"]:
        break
base.close()
del base
grid = json.loads(a.grid)
if isinstance(grid, list):
    combos = grid
else:
    keys = list(grid)
    combos = [dict(zip(keys, vals)) for vals in itertools.product(*[grid[k] for k in keys])]
for kw in combos:
    ctx = SeaIce(cfg.n, **kw)
    ctx.set_step(cfg.dt, cfg.dt, h, A, v0, va, vo)
    out = []
    for l, (vv, pi) in states.items():
        ctx.set_pi(pi)
        R, _ = ctx.residual(vv)
        ctx.assemble_jacobian(vv, pi, want_csr=False)
        torch.cuda.synchronize()
        t0 = time.time()
        nl, oc = ctx.amg_setup()
        torch.cuda.synchronize()
        t1 = time.time()
        x, st, rc = ctx.fgmres(R)
        torch.cuda.synchronize()
        t2 = time.time()
        out.append(f"it{l}: {st['iters']:3d} its L{nl} oc{oc:.2f} setup {1e3*(t1-t0):6.1f} ms solve {1e3*(t2-t1):7.1f} ms")
    print(kw, " | ".join(out), flush=True)
    ctx.close()
    del ctx
    torch.cuda.empty_cache()
