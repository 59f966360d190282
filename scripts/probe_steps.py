"""Probe: solve the first few implicit steps of a config on the GPU and print per-step
Newton/Krylov counts, phase times and the AMG hierarchy (development aid)."""
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
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--newton-log", action="store_true")
ap.add_argument("--params", default="{}")
a = ap.parse_args()
cfg = wl.CONFIGS[a.config]
over = json.loads(a.params)
ctx = SeaIce(cfg.n, **over)
h, A = wl.ice_fields(cfg)
v = ctx.zeros(ctx.N)
vo = wl.ocean_nodal(cfg.n)
for s in range(a.steps):
    t_new = (s + 1) * cfg.dt
    va = wl.wind_nodal(cfg.n, t_new, cfg.moving)
    torch.cuda.synchronize()
    t0 = time.time()
    if a.newton_log:
        ctx.set_step(cfg.dt, t_new, h, A, v, va, vo)
        vv = v.clone()
        recs = []
        for l in range(201):
            d = ctx.newton_step(vv)
            recs.append(d)
            if d["converged_on_entry"]:
                break
            print(f"  it {l:3d} |R|/r0={d['res_norm']/d['res_norm0']:.3e} alpha={d['alpha']:.4g} kry={d['krylov']['iters']:3d}"
                  f" conv={d['krylov']['converged']} lv={d['amg_levels']} oc={d['amg_op_complexity']:.2f}"
                  f" t_asm={d['t_assemble']:.1f} t_amg={d['t_amg']:.1f} t_kry={d['t_krylov']:.1f} t_ls={d['t_ls']:.1f} ms", flush=True)
        v = vv
        print(f"step {s}: newton={len(recs)-1} wall={time.time()-t0:.2f}s", flush=True)
    else:
        vout, st = ctx.solve_step(cfg.dt, t_new, h, A, v, va, vo)
        v = vout
        print(f"step {s}: {json.dumps({k: (round(x, 3) if isinstance(x, float) else x) for k, x in st.items()})}", flush=True)
print("mem live/peak GB", [x / 1e9 for x in ctx.memory()])
