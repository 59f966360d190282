"""Config 3 (n = 1024, 8 moving-cyclone steps) on the GPU product path, with the bulk-viscosity
spread of each converged step (SURVEY reading G25: report max zeta / min zeta, do not tune the
inputs to reach BASELINE's "> 8 orders").

zeta = P / (2 Delta) at every Gauss point, Delta = sqrt(Delta_min^2 + 2 tau:tau)
(Appendix A of SURVEY: |tau^|^2 = (e11 + e22)^2 / 2 + e^-2 ((e11 - e22)^2 / 2 +
2 e12^2)), strain rates of the Q1 velocity at the 2 x 2 Gauss points, P = P* h exp(-C (1 - A)).
This is an analysis of the solver's OUTPUT (numpy, written from the definitions); nothing here
feeds the solve.

  python scripts/zeta_spread.py [--config 3] [--steps 8] > profiles/r02_cfg3_zeta.jsonl
"""
import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2204_10822_b200 import workloads as wl
from paper_2204_10822_b200.seaice import SeaIce


def zeta_stats(v, h, A, n, prm, L=wl.L_DOMAIN):
    dx = L / n
    s = n + 1
    V = v.reshape(s, s, 2)          # [j][i][c]
    v00, v10 = V[:-1, :-1], V[:-1, 1:]
    v11, v01 = V[1:, 1:], V[1:, :-1]
    P = prm.P_star * h.reshape(n, n) * np.exp(-prm.C * (1.0 - A.reshape(n, n)))
    g = 1.0 / math.sqrt(3.0)
    zmin, zmax, dmax = np.inf, 0.0, 0.0
    for xi in (-g, g):
        for eta in (-g, g):
            # d/dx and d/dy of the bilinear interpolant at (xi, eta) (reference [-1, 1]^2)
            dvx = ((v10 - v00) * (1 - eta) + (v11 - v01) * (1 + eta)) / (2.0 * dx)
            dvy = ((v01 - v00) * (1 - xi) + (v11 - v10) * (1 + xi)) / (2.0 * dx)
            e11, e22 = dvx[..., 0], dvy[..., 1]
            e12 = 0.5 * (dvy[..., 0] + dvx[..., 1])
            t2 = 0.5 * (e11 + e22) ** 2 + (0.5 * (e11 - e22) ** 2 + 2.0 * e12 ** 2) / prm.e ** 2
            D = np.sqrt(prm.delta_min ** 2 + 2.0 * t2)
            z = P / (2.0 * D)
            zmin, zmax, dmax = min(zmin, z.min()), max(zmax, z.max()), max(dmax, D.max())
    return {"zeta_min": float(zmin), "zeta_max": float(zmax), "decades": float(np.log10(zmax / zmin)),
            "delta_max_over_delta_min": float(dmax / prm.delta_min)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--params", default="{}")
    a = ap.parse_args()
    cfg = wl.CONFIGS[a.config]
    prm = wl.PhysParams()
    steps = a.steps or cfg.steps
    h, A = wl.ice_fields(cfg)
    vo = wl.ocean_nodal(cfg.n)
    ctx = SeaIce(cfg.n, **json.loads(a.params))
    v = torch.zeros(ctx.N, dtype=torch.float64, device="cuda")
    for s in range(steps):
        va = wl.wind_nodal(cfg.n, (s + 1) * cfg.dt, cfg.moving)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        v, st = ctx.solve_step(cfg.dt, (s + 1) * cfg.dt, h, A, v, va, vo)
        e1.record()
        torch.cuda.synchronize()
        rec = {"config": a.config, "step": s + 1, "s_per_step": e0.elapsed_time(e1) / 1e3,
               "newton": st["newton_iters"], "krylov": st["krylov_iters_total"], "solves": st["krylov_solves"],
               "capped": st["krylov_capped"], "amg_setups": st["amg_setups"], "converged": st["converged"],
               **zeta_stats(v.cpu().numpy(), h, A, cfg.n, prm)}
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
