"""Stress-velocity Newton loop for one implicit time step (ORACLE).

Test infrastructure only.  Follows PAPER.md in order:
  * v_0 = v^n, pi_0 = tau(v^n)/Delta(v^n)                        (reading G4)
  * solve J(v_l, pi_l) v~ = R(v_l)                               (eq:linearSVNewton)
  * alpha = 1, 1/2, ... while Phi does not decrease                (G12, G14)
  * v_{l+1} = v_l + alpha v~, pi_{l+1} = pi_l + alpha pi~          (eq:tautilde)
  * stop at ||R(v_l)||_2 <= rtol ||R(v_0)||_2 (BASELINE.json 1e-8; the paper uses a
    1e4 reduction), absolute floor 1e-14, maxit 200.
"""
from __future__ import annotations

import numpy as np

from . import krylov
from .model import Problem

# Reading G12b: |DeltaPhi| <= LS_ETA * S (S = sum of |terms|) is indistinguishable from 0 in
# fp64; such a step is accepted iff it reduces ||R||_2 (the paper's residual-based
# backtracking, "results in similar results").
LS_ETA = 1e-12


def solve_step(inp, prm, kind="sv", linsolve="direct", rtol=1e-8, maxit=200,
               ls_max=20, krylov_rtol=1e-8, krylov_maxit=300, restart=60,
               project_pi=False, amg_params=None, record_iterates=False, forcing=0, amg_lag=0,
               amg_reuse=0):
    """forcing = 1: Eisenstat-Walker choice 2 for the Krylov tolerance of each solve (reading
    G29): eta_0 = 0.1, eta_l = 0.9 (|R_l|/|R_{l-1}|)^2, safeguards
    eta_l >= 0.9 eta_{l-1}^2 (if > 0.1) and eta_l >= 0.5 rtol |R_0|/|R_l|, clamped to
    [krylov_rtol, 0.1]; after a line search that found no decrease (stagnation flag) the next
    solve uses krylov_rtol.
    amg_lag = T > 0 (reading G31): at Newton iteration l >= 1 the AMG hierarchy is rebuilt only
    if the previous linear solve needed more than T Krylov iterations; otherwise its coarse
    levels are kept and only the finest level is refreshed from the current Jacobian
    (amg.refresh_finest); a hierarchy built with K = 3 near-nullspace columns because v_l was zero
    is rebuilt as soon as v_l != 0 (nullspace_dim = 4).
    amg_reuse = 1 (reading G32): the first AMG setup of the time step builds the aggregates;
    every later setup of the step keeps them (amg.setup(..., reuse=H)) and recomputes all values
    from the current Jacobian and linearisation point."""
    pb = Problem(inp, prm)
    v = pb.v_prev.copy()
    v[pb.bdof] = 0.0
    pi = pb.pi_consistent(v)
    hist = {"res": [], "alpha": [], "dphi": [], "krylov": [], "halvings": [],
            "stagnated": [], "iterates": []}
    r0 = None
    converged = False
    H = None
    for l in range(maxit + 1):
        R = pb.residual(v)
        nr = float(np.linalg.norm(R))
        hist["res"].append(nr)
        if record_iterates:
            hist["iterates"].append((v.copy(), pi.copy()))
        if r0 is None:
            r0 = nr
            if r0 < 1e-14:
                converged = True
                break
        if nr <= rtol * r0:
            converged = True
            break
        if l == maxit:
            break
        krtol = krylov_rtol
        if forcing == 1:
            eta = 0.1
            if l > 0:
                eta = 0.9 * (nr / hist["res"][-2]) ** 2
                if 0.9 * eta_prev ** 2 > 0.1:
                    eta = max(eta, 0.9 * eta_prev ** 2)
            eta = max(eta, 0.5 * rtol * r0 / nr)
            eta = min(max(eta, krylov_rtol), 0.1)
            if l > 0 and hist["stagnated"][-1]:
                # safeguard: the last line search found no energy decrease (the inexact
                # direction was not a descent direction): solve to the floor tolerance
                eta = krylov_rtol
            eta_prev = eta
            krtol = eta
        pi_j = pi if kind == "sv" else None
        J = pb.jacobian(v, pi_j, kind)
        if linsolve == "direct":
            vt = krylov.sparse_direct_solve(J, R)
            kst = {"iters": 0}
        elif linsolve == "dense":
            vt = krylov.dense_cholesky_solve(J, R)
            kst = {"iters": 0}
        elif linsolve == "jacobi_fgmres":
            vt, kst = krylov.fgmres(lambda x: J @ x, R, krylov.jacobi(J), restart, krtol, krylov_maxit)
        elif linsolve in ("amg_fgmres", "amg_pcg"):
            from . import amg
            # the linearisation point v is the fourth near-nullspace column when
            # amg_params["nullspace_dim"] == 4 (reading G30); ignored otherwise
            ap = amg_params or {}
            # (G31 refinement: a hierarchy built without the v_l column, K = 3 because v_l was 0, is
            # not kept once v_l != 0 and nullspace_dim = 4 asks for the fourth column)
            stale_K = H is not None and H["K"] == 3 and ap.get("nullspace_dim", 4) == 4 and bool(np.any(v))
            if H is None or amg_lag <= 0 or hist["krylov"][-1]["iters"] > amg_lag or stale_K:
                H = amg.setup(J, pb, v=v, reuse=H if amg_reuse else None, **ap)
                hist.setdefault("amg_rebuilt", []).append(True)
                hist.setdefault("amg_reused", []).append(H["reused"])
            else:
                H = amg.refresh_finest(H, J, seed=ap.get("seed", 0), power_iters=ap.get("power_iters", 20))
                hist.setdefault("amg_rebuilt", []).append(False)
            if linsolve == "amg_fgmres":
                vt, kst = krylov.fgmres(lambda x: J @ x, R, lambda r: amg.vcycle(H, r), restart,
                                        krtol, krylov_maxit)
            else:
                vt, kst = krylov.pcg(lambda x: J @ x, R, lambda r: amg.vcycle(H, r), krtol, krylov_maxit)
            kst["levels"] = len(H["levels"])
        else:
            raise ValueError(linsolve)
        hist["krylov"].append(kst)
        alpha, dphi, stag, halv = 1.0, 0.0, True, 0
        for k in range(ls_max + 1):
            alpha = 0.5 ** k
            dphi, S = pb.delta_energy(v, vt, alpha, with_abs=True)
            if dphi < -LS_ETA * S:
                stag = False
                halv = k
                break
            if dphi <= LS_ETA * S and np.linalg.norm(pb.residual(v + alpha * vt)) < nr:
                # energy change below roundoff: residual-based acceptance (reading G12b)
                stag = False
                halv = k
                break
        else:
            halv = ls_max
        hist["alpha"].append(alpha)
        hist["dphi"].append(dphi)
        hist["halvings"].append(halv)
        hist["stagnated"].append(stag)
        if kind == "sv":
            pt = pb.pi_tilde(v, pi, vt)
            pi = pi + alpha * pt
            if project_pi:
                T = pb.pi_to_tensor(pi)
                s = np.maximum(1.0, np.sqrt(2.0 * np.sum(T * T, axis=(-2, -1))))
                pi = pb.pi_from_tensor(T / s[..., None, None])
        v = v + alpha * vt
    hist["newton_iters"] = len(hist["alpha"])
    hist["converged"] = converged
    return v, pi, hist
