"""CPU experiment (development aid, not product): AMG-variant FGMRES/PCG counts at late
sv-Newton iterates, using the oracle's Newton (direct solves) to produce the iterates.

  python scripts/exp_amg_cpu.py --n 128 --iterates 4,8,-1 --variants base,vmode,pcg
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import scipy.sparse as sp

from oracle import amg as OA
from oracle import krylov, newton
from oracle.model import Problem
from paper_2204_10822_b200 import workloads as wl


def mgs_k(Bs, k, tol=1e-8):
    m = Bs.shape[0]
    Q = np.zeros((m, k))
    R = np.zeros((k, k))
    for c in range(k):
        v = Bs[:, c].copy()
        n0 = np.sqrt(v @ v)
        for _ in range(2):
            for j in range(c):
                r = Q[:, j] @ v
                R[j, c] += r
                v = v - r * Q[:, j]
        nv = np.sqrt(v @ v)
        if nv > tol * n0 and nv > 0:
            Q[:, c] = v / nv
            R[c, c] = nv
    return Q, R


def tentative_k(agg, B, b):
    k = B.shape[1]
    nb = agg.size
    na = int(agg.max()) + 1
    order = np.argsort(agg, kind="stable")
    order = order[agg[order] >= 0]
    starts = np.searchsorted(agg[order], np.arange(na + 1))
    rows, cols, vals = [], [], []
    Bc = np.zeros((k * na, k))
    for a in range(na):
        mem = order[starts[a]:starts[a + 1]]
        idx = (b * mem[:, None] + np.arange(b)[None, :]).ravel()
        Q, R = mgs_k(B[idx], k)
        Bc[k * a:k * a + k] = R
        rr = np.repeat(idx, k)
        cc = np.tile(k * a + np.arange(k), idx.size)
        rows.append(rr)
        cols.append(cc)
        vals.append(Q.ravel())
    Pt = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(b * nb, k * na))
    Pt.eliminate_zeros()
    return Pt, Bc, na


def setup_k(J, B, theta=0.04, coarse_max_dof=400, power_iters=20, seed=0, cheb_degree=3, cheb_lower=0.03,
            cheb_upper=1.1, max_levels=25):
    A = J.tocsr()
    b = 2
    levels = []
    k = B.shape[1]
    for lvl in range(max_levels):
        Dinv, _ = OA.block_diag_inv(A, b)
        lev = {"A": A, "b": b, "Dinv": Dinv, "nb": A.shape[0] // b}
        lev["lmax"] = OA.lambda_max(A, Dinv, seed, lvl, power_iters)
        levels.append(lev)
        if A.shape[0] <= coarse_max_dof:
            break
        G = OA.strength(A, b, theta)
        roots, isolated, rounds = OA.mis2(G, seed, lvl, 2)
        agg = OA.aggregate(G, roots, isolated)
        na = int(roots.sum())
        if na == 0 or na > 0.9 * lev["nb"]:
            break
        Pt, Bc, na = tentative_k(agg, B, b)
        omega = 4.0 / (3.0 * lev["lmax"])
        P = (Pt - omega * (Dinv @ (A @ Pt))).tocsr()
        R = P.T.tocsr()
        Ac = (R @ (A @ P)).tocsr()
        d = Ac.diagonal()
        fix = d == 0.0
        if fix.any():
            Ac = (Ac + sp.diags(fix.astype(np.float64))).tocsr()
        lev.update({"P": P, "R": R})
        A, B, b = Ac, Bc, k
    import scipy.linalg as sla
    levels[-1]["chol"] = sla.cho_factor(levels[-1]["A"].toarray(), lower=True)
    return {"levels": levels, "cheb_degree": cheb_degree, "cheb_lower": cheb_lower, "cheb_upper": cheb_upper,
            "op_complexity": sum(l["A"].nnz for l in levels) / levels[0]["A"].nnz}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=128)
    ap.add_argument("--seed", type=int, default=3)
    ap.add_argument("--iterates", default="4,8,-1")
    ap.add_argument("--variants", default="base,vmode")
    ap.add_argument("--theta", type=float, default=0.04)
    a = ap.parse_args()
    prm = wl.PhysParams()
    cfg = wl.Config(f"exp{a.n}", a.n, a.seed, 1, True)
    inp = wl.step_inputs(cfg, 0)
    t0 = time.time()
    v, pi, h = newton.solve_step(inp, prm, linsolve="direct", record_iterates=True)
    print(f"newton {h['newton_iters']} in {time.time() - t0:.1f}s", flush=True)
    pb = Problem(inp, prm)
    its = [int(x) for x in a.iterates.split(",")]
    iters = h["iterates"]
    B0 = OA.level0_nullspace(a.n, pb.L)
    for li in its:
        vv, pp = iters[li]
        R = pb.residual(vv)
        J = pb.jacobian(vv, pp, "sv").tocsr()
        out = []
        for var in a.variants.split(","):
            t1 = time.time()
            if var in ("base", "pcg", "gm100"):
                B = B0
            elif var == "vmode":
                B = np.concatenate([B0, vv[:, None]], axis=1)
                B[pb.bdof] = 0.0 if False else B[pb.bdof]
            elif var == "vmode2":
                X = np.repeat(wl.node_coords(a.n)[0].ravel(), 2) if False else None
                B = np.concatenate([B0, vv[:, None], (J @ vv)[:, None] * 0 + vv[:, None] ** 2], axis=1)
            else:
                raise ValueError(var)
            H = setup_k(J, B, theta=a.theta)
            M = lambda r: OA.vcycle(H, r)
            if var == "pcg":
                x, st = krylov.pcg(lambda x: J @ x, R, M, 1e-8, 2000)
            elif var == "gm100":
                x, st = krylov.fgmres(lambda x: J @ x, R, M, 100, 1e-8, 2000)
            else:
                x, st = krylov.fgmres(lambda x: J @ x, R, M, 30, 1e-8, 2000)
            out.append(f"{var}: {st['iters']} its L{len(H['levels'])} oc{H['op_complexity']:.2f} ({time.time() - t1:.0f}s)")
        print(f"iterate {li}: " + " | ".join(out), flush=True)


if __name__ == "__main__":
    main()
