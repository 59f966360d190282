"""Krylov solvers and direct solves for J v~ = R (ORACLE; test infrastructure).

PAPER.md P:983-986 uses FGMRES ("flexible generalized minimum residual")
preconditioned by AMG; P:732-735 uses a sparse direct solver (MUMPS, out of
scope: replaced here by a dense Cholesky / scipy sparse direct solve on tiny
meshes).  The paper does not state the Krylov tolerance or restart (reading
G13): rtol 1e-8 relative to ||b||, restart 60, maxit 300 (restart 30, PETSc's default,
until round 2: the late solves of a time step need 100-160 iterations and lose their
superlinear phase at every restart; stored goldens name the restart they were made with).

FGMRES definition shared (as a definition, not code) with the CUDA path:
right preconditioning, x0 = 0, classical Gram-Schmidt (one pass, PETSc's
default), Givens rotations, inner stop when |g_{j+1}| <= rtol ||b||, explicit
residual r = b - A x at every restart; converged only when that explicit residual
satisfies ||r|| <= rtol ||b|| (an estimate below tol with a larger true residual --
loss of orthogonality in one-pass CGS -- restarts); the iteration count is the total
number of preconditioned matrix-vector products.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla


def fgmres(Aop, b, Mop=None, restart=60, rtol=1e-8, maxit=300):
    b = np.asarray(b, dtype=np.float64)
    N = b.size
    x = np.zeros(N)
    bnorm = float(np.linalg.norm(b))
    stats = {"iters": 0, "restarts": 0, "relres_est": 0.0, "converged": True}
    if bnorm == 0.0:
        return x, stats
    Mop = Mop or (lambda r: r.copy())
    r = b.copy()
    beta = bnorm
    its = 0
    while True:
        V = np.zeros((restart + 1, N))
        Z = np.zeros((restart, N))
        H = np.zeros((restart + 1, restart))
        cs = np.zeros(restart)
        sn = np.zeros(restart)
        g = np.zeros(restart + 1)
        g[0] = beta
        V[0] = r / beta
        j_done = 0
        est = beta
        for j in range(restart):
            Z[j] = Mop(V[j])
            w = Aop(Z[j])
            h = V[: j + 1] @ w                      # classical Gram-Schmidt
            w = w - h @ V[: j + 1]
            hn = float(np.linalg.norm(w))
            H[: j + 1, j] = h
            H[j + 1, j] = hn
            if hn > 0.0:
                V[j + 1] = w / hn
            for i in range(j):                      # previous rotations
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            den = float(np.hypot(H[j, j], H[j + 1, j]))
            cs[j] = H[j, j] / den
            sn[j] = H[j + 1, j] / den
            H[j, j] = den
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            its += 1
            j_done = j + 1
            est = abs(g[j + 1])
            if est <= rtol * bnorm or hn == 0.0 or its >= maxit:
                break
        y = sla.solve_triangular(H[:j_done, :j_done], g[:j_done])
        x = x + y @ Z[:j_done]
        r = b - Aop(x)
        beta = float(np.linalg.norm(r))
        stats["relres_est"] = est / bnorm
        if beta <= rtol * bnorm:
            break
        if its >= maxit:
            stats["converged"] = False
            break
        stats["restarts"] += 1
    stats["iters"] = its
    stats["relres_true"] = beta / bnorm
    return x, stats


def pcg(Aop, b, Mop=None, rtol=1e-8, maxit=5000):
    """Preconditioned conjugate gradients (textbook), x0 = 0; stop when the recursively updated
    residual meets ||r|| <= rtol ||b||.  As for fgmres, convergence is declared only when the
    explicit residual ||b - A x|| also meets it; otherwise CG restarts from that residual."""
    Mop = Mop or (lambda r: r.copy())
    x = np.zeros_like(b)
    bn = float(np.linalg.norm(b))
    its = 0
    if bn == 0.0:
        return x, {"iters": 0, "converged": True, "restarts": 0}
    r = b.copy()
    restarts = 0
    while True:
        z = Mop(r)
        p = z.copy()
        rz = float(r @ z)
        while its < maxit:
            Ap = Aop(p)
            a = rz / float(p @ Ap)
            x += a * p
            r -= a * Ap
            its += 1
            if np.linalg.norm(r) <= rtol * bn:
                break
            z = Mop(r)
            rz_new = float(r @ z)
            p = z + (rz_new / rz) * p
            rz = rz_new
        r = b - Aop(x)
        rn = float(np.linalg.norm(r))
        if rn <= rtol * bn:
            return x, {"iters": its, "converged": True, "restarts": restarts, "relres_true": rn / bn}
        if its >= maxit:
            return x, {"iters": its, "converged": False, "restarts": restarts, "relres_true": rn / bn}
        restarts += 1


def jacobi(J):
    d = J.diagonal().copy()
    return lambda r: r / d


def dense_cholesky_solve(J, b):
    """Dense Cholesky solve (tiny meshes; stands in for the paper's direct solver)."""
    A = J.toarray() if hasattr(J, "toarray") else np.asarray(J)
    c = sla.cho_factor(A, lower=True)
    return sla.cho_solve(c, b)


def sparse_direct_solve(J, b):
    import scipy.sparse.linalg as spla
    return spla.spsolve(J.tocsc(), b)
