"""CPU pins of oracle/amg.py (the AMG definition shared with the GPU path) by
properties the algebra fixes, independent of the oracle's own formulas: MIS(2) independence at
distance 2 and maximality; one aggregate per non-isolated node; orthonormal tentative columns that
reproduce the near-nullspace; SPD Galerkin operators whose energy equals the fine energy of the
prolongated vector; the Chebyshev error polynomial in closed form; a symmetric V-cycle; and an
exact solve when the hierarchy has a single level (checked against an LU solve)."""
import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from oracle import amg
from oracle import model as M
from paper_2204_10822_b200 import workloads as wl

PRM = wl.PhysParams()


def _jacobian(n, seed=5, amp=0.05):
    _, inp = wl.custom_inputs(n, seed=seed)
    pb = M.Problem(inp, PRM)
    v = wl.random_velocity(n, seed + 1, amp=amp)
    pi = wl.random_pi(n, seed + 2)
    return pb, pb.jacobian(v, pi, "sv").tocsr()


@pytest.fixture(scope="module")
def hier():
    pb, J = _jacobian(24)
    return pb, J, amg.setup(J, pb, coarse_max_dof=60, nullspace_dim=3)


def test_mis2_is_distance2_independent_and_maximal():
    pb, J = _jacobian(20)
    G = amg.strength(J, 2, 0.04)
    roots, isolated, _ = amg.mis2(G, 0, 0)
    C = (G + sp.identity(G.shape[0], format="csr")).tocsr()
    C2 = (C @ C).tocsr()  # distance <= 2 reachability
    R = np.where(roots)[0]
    sub = C2[R][:, R].tocoo()
    assert np.all(sub.row == sub.col), "two roots within distance 2"
    covered = np.asarray(C2[:, R].sum(axis=1)).ravel() > 0
    assert np.all(covered | isolated), "a non-isolated node is farther than 2 from every root"


def test_aggregates_partition_non_isolated_nodes():
    pb, J = _jacobian(20)
    G = amg.strength(J, 2, 0.04)
    roots, isolated, _ = amg.mis2(G, 0, 0)
    agg = amg.aggregate(G, roots, isolated)
    assert np.all(agg[~isolated] >= 0) and np.all(agg[isolated] == -1)
    assert np.array_equal(np.sort(np.unique(agg[roots])), np.arange(int(roots.sum())))
    # each root heads its own aggregate
    assert np.array_equal(agg[roots], np.arange(int(roots.sum())))


def test_tentative_orthonormal_and_reproduces_nullspace(hier):
    pb, J, H = hier
    lev = H["levels"][0]
    Pt = lev["Ptent"].toarray()
    PtP = Pt.T @ Pt
    d = np.diag(PtP)
    keep = d > 0.5  # dropped (singular) columns are zero
    assert np.allclose(PtP[np.ix_(keep, keep)], np.eye(keep.sum()), atol=1e-13)
    B = amg.level0_nullspace(pb.n, pb.L)
    # P_tent B_c = B on aggregated rows (isolated rows are zero rows of P_tent)
    Pt_s, Bc, _ = amg.tentative(lev["agg"], B, 2)
    rows = np.repeat(lev["agg"] >= 0, 2)
    assert np.allclose((Pt_s @ Bc)[rows], B[rows], atol=1e-12)


def test_galerkin_operators_spd_and_energy_consistent(hier):
    pb, J, H = hier
    rng = np.random.default_rng(0)
    for l in range(len(H["levels"]) - 1):
        A, P, Ac = H["levels"][l]["A"], H["levels"][l]["P"], H["levels"][l + 1]["A"]
        Acd = Ac.toarray()
        assert np.allclose(Acd, Acd.T, rtol=0, atol=1e-12 * np.abs(Acd).max())
        assert np.linalg.eigvalsh(0.5 * (Acd + Acd.T)).min() > 0
        for _ in range(3):
            xc = rng.standard_normal(Ac.shape[0])
            xf = P @ xc
            ef, ec = xf @ (A @ xf), xc @ (Ac @ xc)
            assert abs(ef - ec) <= 1e-11 * abs(ef)


def test_chebyshev_error_polynomial_closed_form():
    """On a diagonal A with Dinv = I the Chebyshev smoother started from x = 0 gives
    x = (1 - p(lambda)) b / lambda with p(t) = T_m((th - t)/de) / T_m(th/de) (Saad, Alg. 12.1)."""
    lam = np.linspace(0.05, 2.0, 40)
    A = sp.diags(lam).tocsr()
    lev = {"A": A, "Dinv": sp.identity(lam.size, format="csr"), "lmax": lam.max()}
    b = np.ones(lam.size)
    lo, up = 0.03, 1.1
    for m in (1, 2, 3, 5):
        x, r = amg.chebyshev(lev, b, None, m, lo, up, need_residual=True)
        bmax = up * lam.max()
        amin = lo * bmax
        th, de = 0.5 * (bmax + amin), 0.5 * (bmax - amin)
        T = np.polynomial.chebyshev.Chebyshev.basis(m)
        p = T((th - lam) / de) / T(th / de)
        assert np.allclose(x, (1.0 - p) / lam, rtol=1e-12, atol=1e-14)
        assert np.allclose(r, b - lam * x, rtol=1e-12, atol=1e-14)


def test_vcycle_symmetric(hier):
    pb, J, H = hier
    rng = np.random.default_rng(1)
    r1, r2 = rng.standard_normal(J.shape[0]), rng.standard_normal(J.shape[0])
    a, b = amg.vcycle(H, r1) @ r2, r1 @ amg.vcycle(H, r2)
    assert abs(a - b) <= 1e-11 * max(abs(a), abs(b))


def test_single_level_vcycle_is_exact_solve():
    pb, J = _jacobian(8)
    H = amg.setup(J, pb, coarse_max_dof=10 ** 6, nullspace_dim=3)
    assert len(H["levels"]) == 1
    r = np.random.default_rng(2).standard_normal(J.shape[0])
    x = amg.vcycle(H, r)
    xd = spla.splu(J.tocsc()).solve(r)
    assert np.linalg.norm(x - xd) <= 1e-10 * np.linalg.norm(xd)


def _block_eigs_DinvA(J, b):
    """Eigenvalues of D^-1 A (D = b x b block diagonal) by a dense generalized symmetric
    eigen-solve A x = lambda D x (A, D SPD): scipy.linalg.eigh, independent of the oracle."""
    import scipy.linalg as sla
    A = J.toarray()
    D = np.zeros_like(A)
    for I in range(A.shape[0] // b):
        s = slice(b * I, b * I + b)
        D[s, s] = A[s, s]
    return sla.eigh(A, D, eigvals_only=True)


@pytest.mark.parametrize("n,seed", [(8, 3), (12, 4)])
def test_lambda_max_power_iteration_vs_eigensolve(n, seed):
    """lambda_max (20 power iterations on D^-1 A from the seeded start) lies within
    [0.9, 1.0] x the largest eigenvalue of the pencil (A, D) from a dense eigen-solve.  It feeds
    omega = 4/(3 lambda) and the Chebyshev interval [lo b, b], b = 1.1 lambda."""
    pb, J = _jacobian(n, seed=seed)
    Dinv, _ = amg.block_diag_inv(J, 2)
    lam = amg.lambda_max(J, Dinv, 0, 0, 20)
    ev = _block_eigs_DinvA(J, 2)
    assert 0.9 * ev.max() <= lam <= 1.0 * ev.max() * (1 + 1e-12), (lam, ev.max())


def test_strength_threshold_hand_example():
    """DESIGN §5 strength: blocks I != J strong iff ||A_IJ||_F^2 >= theta^2 ||A_II||_F ||A_JJ||_F.
    Three nodes, A_00 = 2 I, A_11 = 8 I, A_22 = 8 I, A_01 = c I, A_12 = 0.5 I: ||A_01||^2 = 2 c^2
    against theta^2 * (2 sqrt2)(8 sqrt2) = 32 theta^2, so with theta = 0.25 the pair (0,1) is
    strong iff c >= 1 (checked just above and below); (1,2): 2 * 0.25 = 0.5 < 0.0625 * 128 = 8, weak.
    The stored strength value is s_IJ = ||A_IJ||^2 / (||A_II|| ||A_JJ||)."""
    for c, strong in ((1.001, True), (0.999, False), (1.3, True)):
        blocks = {(0, 0): 2.0, (1, 1): 8.0, (2, 2): 8.0, (0, 1): c, (1, 0): c, (1, 2): 0.5, (2, 1): 0.5}
        A = np.zeros((6, 6))
        for (I, K), s in blocks.items():
            A[2 * I:2 * I + 2, 2 * K:2 * K + 2] = s * np.eye(2)
        G = amg.strength(sp.csr_matrix(A), 2, 0.25).toarray()
        assert (G[0, 1] > 0) == strong and (G[1, 0] > 0) == strong
        assert G[1, 2] == 0 and G[2, 1] == 0
        if strong:
            assert abs(G[0, 1] - 2 * c * c / 32.0) <= 1e-15


def test_v_column_is_near_null_for_the_plastic_part_and_reproduced_by_ptent():
    """Reading G30 (nullspace_dim = 4).  (a) The fact that justifies the fourth column: at a
    consistent pi = tau(v)/Delta(v) the sv coefficient maps tau(v) to (P/Delta)(Delta_min^2 /
    Delta^2) tau(v) (eq:modification), so the viscous part of J annihilates v up to
    that factor while the Picard part (P/Delta) I does not.  Checked on the assembled operators at
    a small plastic velocity (strain >> Delta_min, mass and drag energies negligible): v's energy
    under J_sv is a few % of its Picard energy, while an independent random field keeps > 30 %.
    (b) P_tent B_c = [rigid modes, v] exactly on aggregated rows, columns orthonormal."""
    n = 24
    _, inp = wl.custom_inputs(n, seed=5)
    pb = M.Problem(inp, PRM)
    v = wl.random_velocity(n, 6, amp=0.005)
    w = wl.random_velocity(n, 7, amp=0.005)
    pi = pb.pi_consistent(v)
    Jsv = pb.jacobian(v, pi, "sv").tocsr()
    Jpi = pb.jacobian(v, None, "picard").tocsr()
    # energies of v: Picard viscous part E_p = v^T (Jpi - M - D) v > 0; sv removes all but
    # a Delta_min^2/Delta^2 fraction of it
    Ep = v @ (Jpi @ v)
    Es = v @ (Jsv @ v)
    assert 0 < Es < 0.05 * Ep
    assert w @ (Jsv @ w) > 0.3 * (w @ (Jpi @ w))
    H = amg.setup(Jsv, pb, v=v, nullspace_dim=4, coarse_max_dof=60)
    lev = H["levels"][0]
    B = amg.level0_nullspace(pb.n, pb.L, v)
    assert B.shape[1] == 4
    Pt_s, Bc, _ = amg.tentative(lev["agg"], B, 2)
    rows = np.repeat(lev["agg"] >= 0, 2)
    assert np.allclose((Pt_s @ Bc)[rows], B[rows], atol=1e-12 * np.abs(B).max())
    PtP = (Pt_s.T @ Pt_s).toarray()
    keep = np.diag(PtP) > 0.5
    assert np.allclose(PtP[np.ix_(keep, keep)], np.eye(keep.sum()), atol=1e-13)
    # coarse blocks are 4 x 4 and the Galerkin operator is SPD
    Ac = H["levels"][1]["A"].toarray()
    assert Ac.shape[0] % 4 == 0
    assert np.linalg.eigvalsh(0.5 * (Ac + Ac.T)).min() > 0


def test_refresh_finest_keeps_coarse_levels_and_symmetry():
    """Reading G31: the lagged hierarchy replaces only the finest operator (and its D^-1,
    lambda_max); the coarse levels are those of the old hierarchy, and the V-cycle stays
    symmetric (so it remains a valid SPD preconditioner for the new J)."""
    pb, J = _jacobian(24, seed=5)
    _, J2 = _jacobian(24, seed=9)
    v = wl.random_velocity(24, 6, amp=0.05)
    H = amg.setup(J, pb, v=v, coarse_max_dof=60)
    H2 = amg.refresh_finest(H, J2)
    assert H2["levels"][0]["A"] is not H["levels"][0]["A"]
    assert abs(H2["levels"][0]["A"] - J2).max() == 0
    for l in range(1, len(H["levels"])):
        assert H2["levels"][l] is H["levels"][l]
    assert H2["levels"][0]["P"] is H["levels"][0]["P"]
    rng = np.random.default_rng(1)
    r1, r2 = rng.standard_normal(J.shape[0]), rng.standard_normal(J.shape[0])
    z1, z2 = amg.vcycle(H2, r1), amg.vcycle(H2, r2)
    assert abs(z1 @ r2 - r1 @ z2) <= 1e-10 * abs(z1 @ r2)


@pytest.mark.parametrize("dist", [1, 3])
def test_misd_is_distance_d_independent_and_maximal(dist):
    """MIS(d) for the agg_dist options: no two roots within graph distance d, every non-isolated
    node within distance d of a root (brute-force reachability by powers of the closed graph)."""
    pb, J = _jacobian(20)
    G = amg.strength(J, 2, 0.04)
    roots, isolated, _ = amg.mis2(G, 0, 0, dist=dist)
    C = (G + sp.identity(G.shape[0], format="csr")).tocsr()
    Cd = C.copy()
    for _ in range(dist - 1):
        Cd = (Cd @ C).tocsr()
    R = np.where(roots)[0]
    sub = Cd[R][:, R].tocoo()
    assert np.all(sub.row == sub.col), f"two roots within distance {dist}"
    covered = np.asarray(Cd[:, R].sum(axis=1)).ravel() > 0
    assert np.all(covered | isolated)


def test_reused_aggregates_hierarchy_is_galerkin_for_the_new_operator():
    """Reading G32 (amg.setup(..., reuse=H)): with the aggregates of a hierarchy built for one
    (J1, v1), the hierarchy for another (J2, v2) keeps every level's aggregates and the level
    count, its tentative prolongators reproduce the NEW near-nullspace [rigid modes, v2] exactly,
    its coarse operators are P^T A P of the new operator (checked densely, not through the
    oracle's own product order), and reusing a hierarchy's own aggregates reproduces it."""
    n = 20
    _, inp = wl.custom_inputs(n, seed=5)
    pb = M.Problem(inp, PRM)
    v1 = wl.random_velocity(n, 6, amp=0.05)
    v2 = wl.random_velocity(n, 9, amp=0.03)
    J1 = pb.jacobian(v1, pb.pi_consistent(v1), "sv").tocsr()
    J2 = pb.jacobian(v2, pb.pi_consistent(v2), "sv").tocsr()
    H1 = amg.setup(J1, pb, v=v1, coarse_max_dof=60)
    H2 = amg.setup(J2, pb, v=v2, coarse_max_dof=60, reuse=H1)
    assert H2["reused"] and len(H2["levels"]) == len(H1["levels"]) >= 3
    Bl = amg.level0_nullspace(n, pb.L, v2)
    b = 2
    for l1, l2 in zip(H1["levels"][:-1], H2["levels"][:-1]):
        assert np.array_equal(l1["agg"], l2["agg"])
        Pt = l2["Ptent"].toarray()
        rows = np.repeat(l2["agg"] >= 0, b)  # isolated rows are zero rows of P_tent
        # P_tent has orthonormal columns and spans the level's (new) near-nullspace on aggregated rows
        PtP = Pt.T @ Pt
        keep = np.diag(PtP) > 0.5
        assert np.allclose(PtP[np.ix_(keep, keep)], np.eye(keep.sum()), atol=1e-12)
        coef, *_ = np.linalg.lstsq(Pt[rows], Bl[rows], rcond=None)
        assert np.linalg.norm(Pt[rows] @ coef - Bl[rows]) <= 1e-10 * np.linalg.norm(Bl[rows])
        Bl, b = coef, Bl.shape[1]
    for l, lev in enumerate(H2["levels"][:-1]):
        A = lev["A"].toarray()
        P = lev["P"].toarray()
        Ac = H2["levels"][l + 1]["A"].toarray()
        d = np.diag(Ac).copy()
        ref = P.T @ A @ P
        fix = np.diag(ref) == 0.0
        ref[np.diag_indices_from(ref)] += fix.astype(float)
        assert np.abs(Ac - ref).max() <= 1e-10 * np.abs(ref).max(), l
        assert np.all(d > 0)
    assert np.abs(H2["levels"][0]["A"] - J2).max() == 0.0
    H1b = amg.setup(J1, pb, v=v1, coarse_max_dof=60, reuse=H1)
    for a, b in zip(H1["levels"], H1b["levels"]):
        assert abs(a["A"] - b["A"]).max() == 0.0 and a["lmax"] == b["lmax"]
    # a different near-nullspace dimension falls back to a full setup
    H3 = amg.setup(J2, pb, v=np.zeros_like(v2), coarse_max_dof=60, reuse=H1)
    assert not H3["reused"]
