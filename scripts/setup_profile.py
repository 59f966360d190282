"""AMG setup phase breakdown under bench conditions (dev aid).

Runs config 4 time steps with SEAICE_SETUP_TIMING=1 (set by this script before the library
loads) and aggregates the per-phase wall times the library prints (synchronising ticks) over
the setups of the last --steps steps.

  python scripts/setup_profile.py --steps 1 --warmup 3 [--params '{...}']
"""
import argparse
import collections
import json
import os
import re
import sys
import tempfile

os.environ["SEAICE_SETUP_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2204_10822_b200 import workloads as wl
from paper_2204_10822_b200.seaice import SeaIce

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--params", default="{}")
a = ap.parse_args()
cfg = wl.CONFIGS[a.config]
h, A = wl.ice_fields(cfg)
vo = wl.ocean_nodal(cfg.n)
ctx = SeaIce(cfg.n, **json.loads(a.params))
v = torch.zeros(ctx.N, dtype=torch.float64, device="cuda")
# redirect fd 2 to a file so the library's fprintf(stderr) lines can be parsed
tmp = tempfile.NamedTemporaryFile(delete=False)
saved = os.dup(2)
os.dup2(tmp.fileno(), 2)
marks = []
for s in range(a.warmup + a.steps):
    va = wl.wind_nodal(cfg.n, (s + 1) * cfg.dt, cfg.moving)
    sys.stderr.flush()
    marks.append(os.lseek(tmp.fileno(), 0, os.SEEK_CUR))
    v, st = ctx.solve_step(cfg.dt, (s + 1) * cfg.dt, h, A, v, va, vo)
    torch.cuda.synchronize()
    if s >= a.warmup:
        print(f"step {s + 1}: newton {st['newton_iters']} krylov {st['krylov_iters_total']} "
              f"t_amg {st['t_amg']:.1f} ms t_krylov {st['t_krylov']:.1f} ms", flush=True)
os.dup2(saved, 2)
txt = open(tmp.name).read()[marks[a.warmup]:] if False else open(tmp.name).read()
lines = txt.splitlines()
# keep only the lines of the timed steps (after the warmup marker)
with open(tmp.name, "rb") as f:
    f.seek(marks[a.warmup])
    lines = f.read().decode(errors="replace").splitlines()
tot = collections.defaultdict(float)
nset = 0
for ln in lines:
    m = re.match(r"\[setup\] L(\d+)\s+(.+?)\s+([\d.]+) ms", ln)
    if not m:
        continue
    lvl, what, ms = m.group(1), m.group(2).strip(), float(m.group(3))
    # SpGEMM ticks carry the product's row count, not a level: keyed by its order of magnitude
    key = f"{what} rows~1e{len(lvl) - 1}" if what.startswith("sg.") else f"L{lvl} {what}"
    tot[key] += ms
    if what == "graph_free":
        nset += 1
print(f"setups: {nset}")
for k, ms in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"  {k:24s} {ms / max(nset, 1):8.2f} ms/setup")
print(f"  total {sum(tot.values()) / max(nset, 1):.1f} ms/setup")
