"""Smoothed-aggregation AMG preconditioner — serial reference of the DEFINITION the GPU
implements (ORACLE tier B; test infrastructure only).

The paper preconditions FGMRES with hypre BoomerAMG (classical coarsening,
strong threshold 0.5, 3 smoothing steps).  BASELINE.json mandates instead an aggregation
AMG with Chebyshev-Jacobi smoothing built on the GPU, so the algorithm below is a
DESIGN.md definition (reading G15-G17), not a paper result.  Parity of the hierarchy
SHAPE (levels, aggregate counts) is therefore "parity unpinned": only its algebra is
pinned (Galerkin identity, P_tent orthonormality and near-nullspace reproduction,
single-level exactness, V-cycle symmetry, Chebyshev closed form).

Definition (every choice is a parameter; both sides implement it independently):
  strength   node blocks I != J strong iff ||A_IJ||_F^2 >= theta^2 ||A_II||_F ||A_JJ||_F and
             ||A_IJ|| > 0; a node with no strong neighbour is isolated (zero P row).
  MIS(2)     tuples (state, hash, index) packed in a uint64 key, state IN=2 > UNDECIDED=1
             > OUT=0, hash = top 37 bits of splitmix64(index + GOLDEN*(64 seed + level + 1)),
             index in 25 bits.  Round: T1 = closed-neighbourhood max of T0, T2 = that of T1;
             UNDECIDED i becomes IN if T2 == T0 (its own key), else OUT if state(T2) == IN.
  aggregates roots numbered in index order; phase 1: a non-root joins the root among its
             strong neighbours with the largest s_IJ = ||A_IJ||^2/(||A_II|| ||A_JJ||), ties to the
             smaller aggregate id; phase 2: the same rule over neighbours assigned in phase 1;
             phase 3: the same over neighbours assigned in phase 2; else unaggregated.
  P_tent     per aggregate (members in index order) modified Gram-Schmidt, two projection
             passes, of the stacked near-nullspace rows; a column whose remaining norm is
             <= 1e-8 of its original norm is dropped (zero column); B_c = R.
             Level-0 near-nullspace: (1,0), (0,1), (-(y - L/2), x - L/2)/L per node, and with
             nullspace_dim = 4 (reading G30) the linearisation point v_l as a fourth column.
  smoothing  P = P_tent - omega D^-1 A P_tent, omega = 4/(3 lambda), D = block diagonal.
  lambda     power iteration on D^-1 A, `power_iters` steps from x0_i = uniform[-1,1) drawn
             by splitmix64(i + GOLDEN*(64 seed + level + 7)); lambda = ||D^-1 A x|| for ||x|| = 1.
  coarse op  A_c = P^T (A P); coarse DOFs whose diagonal is exactly 0 (dropped columns) get 1.
  recursion  stop when 3 n_agg <= coarse_max_dof, at max_levels, or when n_agg > 0.9 n_nodes.
  coarsest   dense Cholesky solve.
  reuse      (reading G32, `reuse=H_prev`) the aggregates of H_prev are kept level by level (no
             strength graph / MIS / aggregation; same level count), everything else — near-
             nullspace with the current v, P_tent, lambda, smoothed P, Galerkin operators,
             coarse factor — is recomputed from the current J.  Ignored (full setup) when the
             near-nullspace dimension differs from H_prev's.
  smoother   Chebyshev of degree m for D^-1 A on [lo b, b], b = up * lambda (Saad Alg. 12.1):
             th = (b+a)/2, de = (b-a)/2, sg = th/de, rho = 1/sg, d = D^-1 r/th;
             repeat m times: x += d; r -= A d; rho' = 1/(2 sg - rho); d = rho' rho d + 2 rho'/de D^-1 r.
  V-cycle    pre-smooth from 0, restrict r, recurse, prolong-add, post-smooth (same polynomial).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M64 = (1 << 64) - 1


def splitmix64(x):
    """Steele et al. splitmix64 finaliser (uint64 in, uint64 out, wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = np.asarray(x, dtype=np.uint64) + GOLDEN
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _salt(seed, level, extra):
    with np.errstate(over="ignore"):
        return GOLDEN * np.uint64(64 * seed + level + extra)


def node_hash(nb, seed, level):
    idx = np.arange(nb, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return splitmix64(idx + _salt(seed, level, 1)) >> np.uint64(27)


def power_start(N, seed, level):
    idx = np.arange(N, dtype=np.uint64)
    with np.errstate(over="ignore"):
        u = (splitmix64(idx + _salt(seed, level, 7)) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return 2.0 * u - 1.0


def block_norms2(A, b):
    """Squared Frobenius norms of the b x b blocks of scalar CSR A -> node-level CSR."""
    N = A.shape[0]
    nb = N // b
    S = sp.csr_matrix((np.ones(N), (np.arange(N), np.arange(N) // b)), shape=(N, nb))
    A2 = A.multiply(A).tocsr()
    F2 = (S.T @ A2 @ S).tocsr()
    F2.sort_indices()
    return F2


def strength(A, b, theta):
    F2 = block_norms2(A, b)
    d = np.sqrt(F2.diagonal())
    F2 = F2.tocoo()
    i, j, f2 = F2.row, F2.col, F2.data
    strong = (i != j) & (f2 > 0) & (f2 >= theta * theta * d[i] * d[j])
    nb = A.shape[0] // b
    sval = np.where(strong, f2 / np.maximum(d[i] * d[j], 1e-300), 0.0)
    G = sp.csr_matrix((sval[strong], (i[strong], j[strong])), shape=(nb, nb))
    G.sort_indices()
    return G


def mis2(G, seed, level, dist=2):
    """Round-synchronous MIS(2) on the strength graph G (definition in the module header);
    dist = d gives MIS(d) (d closed-neighbourhood max passes per round, d = 1..3)."""
    nb = G.shape[0]
    deg = np.diff(G.indptr)
    isolated = deg == 0
    state = np.where(isolated, 0, 1).astype(np.uint64)
    h = node_hash(nb, seed, level)
    idx = np.arange(nb, dtype=np.uint64)
    C = (G + sp.identity(nb, format="csr")).tocsr()       # closed neighbourhoods
    C.sort_indices()
    rounds = 0
    while np.any(state == 1):
        key = (state << np.uint64(62)) | (h << np.uint64(25)) | idx
        T2 = key
        for _ in range(dist):
            T2 = np.maximum.reduceat(T2[C.indices], C.indptr[:-1])
        und = state == 1
        new_in = und & (T2 == key)
        new_out = und & ~new_in & ((T2 >> np.uint64(62)) == 2)
        state = state.copy()
        state[new_in] = 2
        state[new_out] = 0
        rounds += 1
        if rounds > 10000:
            raise RuntimeError("MIS(2) did not terminate")
    return state == 2, isolated, rounds


def aggregate(G, roots, isolated):
    nb = G.shape[0]
    agg = np.full(nb, -1, dtype=np.int64)
    agg[roots] = np.arange(int(roots.sum()))

    def join(assigned_mask, cand_mask):
        Gc = G.tocoo()
        i, j, s = Gc.row, Gc.col, Gc.data
        ok = cand_mask[i] & assigned_mask[j]
        i, j, s = i[ok], j[ok], s[ok]
        if i.size == 0:
            return
        aj = agg[j]
        order = np.lexsort((aj, -s, i))  # by row, then strength desc, then agg id asc
        i, aj = i[order], aj[order]
        first = np.ones(i.size, dtype=bool)
        first[1:] = i[1:] != i[:-1]
        agg[i[first]] = aj[first]

    un = (agg < 0) & ~isolated
    join(roots.copy(), un)                                     # phase 1
    p1 = agg >= 0
    un = (agg < 0) & ~isolated
    join(p1, un)                                               # phase 2
    p2 = agg >= 0
    un = (agg < 0) & ~isolated
    join(p2, un)                                               # phase 3
    return agg


def mgs_qr(Bs, tol=1e-8):
    """Two-pass modified Gram-Schmidt with column dropping; returns Q (m x k), R (k x k)."""
    m, kk = Bs.shape
    Q = np.zeros((m, kk))
    R = np.zeros((kk, kk))
    for k in range(kk):
        v = Bs[:, k].copy()
        n0 = np.sqrt(v @ v)
        for _ in range(2):
            for j in range(k):
                r = Q[:, j] @ v
                R[j, k] += r
                v = v - r * Q[:, j]
        nv = np.sqrt(v @ v)
        if nv > tol * n0 and nv > 0:
            Q[:, k] = v / nv
            R[k, k] = nv
    return Q, R


def tentative(agg, B, b):
    nb = agg.size
    K = B.shape[1]
    na = int(agg.max()) + 1 if agg.size and agg.max() >= 0 else 0
    rows, cols, vals = [], [], []
    Bc = np.zeros((K * na, K))
    members = [[] for _ in range(na)]
    for I in range(nb):
        if agg[I] >= 0:
            members[agg[I]].append(I)
    for a in range(na):
        mem = members[a]
        Bs = np.concatenate([B[b * I:b * I + b] for I in mem], axis=0)
        Q, R = mgs_qr(Bs)
        Bc[K * a:K * a + K] = R
        for t, I in enumerate(mem):
            for r in range(b):
                for k in range(K):
                    rows.append(b * I + r)
                    cols.append(K * a + k)
                    vals.append(Q[t * b + r, k])
    Pt = sp.csr_matrix((vals, (rows, cols)), shape=(b * nb, K * na))
    return Pt, Bc, na


def block_diag_inv(A, b):
    N = A.shape[0]
    nb = N // b
    Ad = A.tocsr()
    blocks = np.zeros((nb, b, b))
    for r in range(b):
        for c in range(b):
            rr = np.arange(nb) * b + r
            cc = np.arange(nb) * b + c
            blocks[:, r, c] = np.asarray(Ad[rr, cc]).ravel()
    inv = np.linalg.inv(blocks)
    Dinv = sp.bsr_matrix((inv, np.arange(nb), np.arange(nb + 1)), shape=(N, N)).tocsr()
    return Dinv, inv


def lambda_max(A, Dinv, seed, level, iters):
    x = power_start(A.shape[0], seed, level)
    x = x / np.linalg.norm(x)
    lam = 0.0
    for _ in range(iters):
        y = Dinv @ (A @ x)
        nrm = np.linalg.norm(y)
        lam = nrm / np.linalg.norm(x)
        x = y / nrm
    return lam


def level0_nullspace(n, L, v=None):
    """Rigid-body modes (1,0), (0,1), (-(y - L/2), x - L/2)/L per node; with v given (reading
    G30) a fourth column: the linearisation point's velocity v_l itself."""
    i = np.arange(n + 1, dtype=np.float64) * (L / n)
    X, Y = np.meshgrid(i, i, indexing="xy")
    X, Y = X.ravel(), Y.ravel()
    Nn = X.size
    B = np.zeros((2 * Nn, 3 if v is None else 4))
    B[0::2, 0] = 1.0
    B[1::2, 1] = 1.0
    B[0::2, 2] = -(Y - 0.5 * L) / L
    B[1::2, 2] = (X - 0.5 * L) / L
    if v is not None:
        B[:, 3] = v
    return B


def setup(J, pb=None, theta=0.04, coarse_max_dof=400, max_levels=25, power_iters=20, seed=0,
          cheb_degree=3, cheb_lower=0.03, cheb_upper=1.1, n=None, L=512e3, agg_dist0=2, agg_dist=3,
          v=None, nullspace_dim=4, reuse=None):
    """nullspace_dim = 4 (reading G30) appends the linearisation point v (required then) to
    the three rigid-body modes; coarse levels then carry 4 x 4 blocks.  If v is identically
    zero the three rigid-body modes are used (3 x 3 coarse blocks)."""
    if pb is not None:
        n, L = pb.n, pb.L
    A = J.tocsr()
    b = 2
    if nullspace_dim == 4 and v is None:
        raise ValueError("nullspace_dim = 4 needs the linearisation point v")
    if nullspace_dim == 4 and not np.any(v):
        nullspace_dim = 3  # reading G30: v_l = 0 (e.g. the first iterate from rest) adds no column
    B = level0_nullspace(n, L, v if nullspace_dim == 4 else None)
    K = B.shape[1]
    if reuse is not None and reuse.get("K") != K:
        reuse = None  # reading G32: a different near-nullspace dimension changes the block size
    keep = reuse["levels"] if reuse is not None else None
    levels = []
    for lvl in range(max_levels):
        Dinv, blocks = block_diag_inv(A, b)
        lev = {"A": A, "b": b, "Dinv": Dinv, "nb": A.shape[0] // b}
        lev["lmax"] = lambda_max(A, Dinv, seed, lvl, power_iters)
        levels.append(lev)
        if keep is not None:
            if lvl == len(keep) - 1:
                break
            agg, roots, rounds = keep[lvl]["agg"], keep[lvl]["roots"], 0
            na = int(roots.sum())
        else:
            if A.shape[0] <= coarse_max_dof or lvl + 1 == max_levels:
                break
            G = strength(A, b, theta)
            roots, isolated, rounds = mis2(G, seed, lvl, agg_dist0 if lvl == 0 else agg_dist)
            agg = aggregate(G, roots, isolated)
            na = int(roots.sum())
            if na == 0 or na > 0.9 * lev["nb"]:
                break
        Pt, Bc, na = tentative(agg, B, b)
        omega = 4.0 / (3.0 * lev["lmax"])
        P = (Pt - omega * (Dinv @ (A @ Pt))).tocsr()
        R = P.T.tocsr()
        Ac = (R @ (A @ P)).tocsr()
        d = Ac.diagonal()
        fix = d == 0.0
        if fix.any():
            Ac = (Ac + sp.diags(fix.astype(np.float64))).tocsr()
        lev.update({"P": P, "R": R, "Ptent": Pt, "agg": agg, "roots": roots, "mis_rounds": rounds, "na": na})
        A, B, b = Ac, Bc, K
    coarse = levels[-1]
    coarse["chol"] = sla.cho_factor(coarse["A"].toarray(), lower=True)
    nnz0 = levels[0]["A"].nnz
    return {"levels": levels, "cheb_degree": cheb_degree, "cheb_lower": cheb_lower, "cheb_upper": cheb_upper,
            "K": K, "reused": keep is not None,
            "op_complexity": sum(l["A"].nnz for l in levels) / nnz0}


def refresh_finest(H, J, seed=0, power_iters=20):
    """Lagged hierarchy (reading G31): keep the coarse levels (P, R, A_l for l >= 1) of H and
    replace only the finest level's operator by the current J, with its block-diagonal inverse
    and lambda_max recomputed (the smoother on level 0 always uses the current Jacobian)."""
    lev0 = dict(H["levels"][0])
    A = J.tocsr()
    Dinv, _ = block_diag_inv(A, lev0["b"])
    lev0.update({"A": A, "Dinv": Dinv, "lmax": lambda_max(A, Dinv, seed, 0, power_iters)})
    levels = [lev0] + H["levels"][1:]
    if len(levels) == 1:
        levels[0]["chol"] = sla.cho_factor(A.toarray(), lower=True)
    return {**H, "levels": levels}


def chebyshev(lev, bvec, x, m, lo, up, need_residual):
    """Chebyshev(m) for D^-1 A on [lo*bmax, bmax], bmax = up*lambda (Saad, Alg. 12.1).
    Returns x and, if need_residual, r = b - A x (from the recurrence)."""
    A, Dinv = lev["A"], lev["Dinv"]
    bmax = up * lev["lmax"]
    amin = lo * bmax
    th = 0.5 * (bmax + amin)
    de = 0.5 * (bmax - amin)
    sg = th / de
    rho = 1.0 / sg
    r = bvec - A @ x if x is not None else bvec.copy()
    x = np.zeros_like(bvec) if x is None else x.copy()
    d = (Dinv @ r) / th
    for k in range(m):
        x = x + d
        if k < m - 1 or need_residual:
            r = r - A @ d
        if k < m - 1:
            rho_new = 1.0 / (2.0 * sg - rho)
            d = rho_new * rho * d + (2.0 * rho_new / de) * (Dinv @ r)
            rho = rho_new
    return x, r


def vcycle(H, bvec, l=0):
    levels = H["levels"]
    lev = levels[l]
    if l == len(levels) - 1:
        return sla.cho_solve(lev["chol"], bvec)
    m, lo, up = H["cheb_degree"], H["cheb_lower"], H["cheb_upper"]
    x, r = chebyshev(lev, bvec, None, m, lo, up, need_residual=True)
    ec = vcycle(H, lev["R"] @ r, l + 1)
    x = x + lev["P"] @ ec
    x, _ = chebyshev(lev, bvec, x, m, lo, up, need_residual=False)
    return x
