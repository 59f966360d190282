"""Micro-benchmark: V-cycle and FGMRES-iteration cost at a late Newton iterate (dev aid).

Builds the hierarchy at sv-Newton iterate --iterate of the config's first step, then times
--reps preconditioner applications (graph path) and prints the per-class profile of one
eager pass."""
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
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--iterate", type=int, default=8)
ap.add_argument("--reps", type=int, default=50)
ap.add_argument("--params", default="{}")
ap.add_argument("--ncu-range", action="store_true", help="wrap one V-cycle in cudaProfilerStart/Stop")
a = ap.parse_args()
cfg = wl.CONFIGS[a.config]
h, A = wl.ice_fields(cfg)
va = wl.wind_nodal(cfg.n, cfg.dt, cfg.moving)
vo = wl.ocean_nodal(cfg.n)
ctx = SeaIce(cfg.n, **json.loads(a.params))
v = torch.zeros(ctx.N, dtype=torch.float64, device="cuda")
ctx.set_step(cfg.dt, cfg.dt, h, A, v, va, vo)
for l in range(a.iterate):
    ctx.newton_step(v)
ctx.assemble_jacobian(v, None, want_csr=False)
torch.cuda.synchronize()
t0 = time.time()
nl, oc = ctx.amg_setup()
torch.cuda.synchronize()
print(f"setup {1e3*(time.time()-t0):.1f} ms levels {nl} oc {oc:.3f}")
for l in range(nl):
    Al, _, _ = ctx.amg_level(l)
    print(f"  level {l}: block rows {Al['nbrows']} b {Al['br']} nnzb {Al['col_idx'].numel()} "
          f"blocks/row {Al['col_idx'].numel()/Al['nbrows']:.1f}")
r = torch.randn(ctx.N, dtype=torch.float64, device="cuda")
z = ctx.precond_apply(r)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(3):
    ctx.precond_apply(r)
e0.record()
for _ in range(a.reps):
    ctx.precond_apply(r)
e1.record()
torch.cuda.synchronize()
print(f"V-cycle (graph, incl. API sync): {e0.elapsed_time(e1)/a.reps*1e3:.1f} us")
ctx.profile(True)
for _ in range(5):
    ctx.precond_apply(r)
p = ctx.profile_read()
ctx.profile(False)
for k, d in p.items():
    if d["launches"]:
        print(f"  {k:14s} {d['ms']/5*1e3:9.1f} us/vcycle  {d['launches']/5:5.1f} launches  "
              f"{d['bytes']/max(d['ms'],1e-9)/1e6:8.1f} GB/s")
if a.ncu_range:
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    ctx.precond_apply(r)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
R, _ = ctx.residual(v)
x, st, rc = ctx.fgmres(R)
torch.cuda.synchronize()
t0 = time.time()
x, st, rc = ctx.fgmres(R)
torch.cuda.synchronize()
dt = time.time() - t0
print(f"FGMRES: {st['iters']} its, {1e3*dt:.1f} ms, {1e3*dt/max(st['iters'],1):.3f} ms/it")
ctx.profile(True)
x, st, rc = ctx.fgmres(R)
p = ctx.profile_read()
ctx.profile(False)
print(f"FGMRES profiled (eager V-cycle): {st['iters']} its")
for k, d in p.items():
    if d["launches"]:
        print(f"  {k:14s} {d['ms']/st['iters']*1e3:9.1f} us/it  {d['launches']/st['iters']:5.1f} launches/it  "
              f"{d['bytes']/max(d['ms'],1e-9)/1e6:8.1f} GB/s")

