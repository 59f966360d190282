"""Pins of the CPU oracle against what the paper and the mathematics fix.

Each test names the passage it pins (P:<line> = /root/reference/PAPER.md line,
read offline; nothing here reads /root/reference at run time).  The oracle is
written in the paper's 2x2-tensor notation; these tests check it against closed
forms, identities, finite differences, hand derivations and brute force, chosen
so that a dropped term, a wrong sign or a transposed operand fails one of them.
"""
import dataclasses
import json
import math
import os

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import fem, krylov, newton
from oracle import model as M
from paper_2204_10822_b200 import workloads as wl

PRM = wl.PhysParams()
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def small_problem(n=8, seed=0, prm=PRM, moving=False):
    cfg, inp = wl.custom_inputs(n, seed=seed, moving=moving)
    return M.Problem(inp, prm), inp


# ------------------------------------------------------------------ Q1 tables
def test_q1_tables_closed_form():
    """Textbook Q1/2x2-Gauss values (reading G3): N_a(q) in {(2+r3)/6, 1/6, (2-r3)/6}."""
    dx = 3.0
    Nq, dN, w = fem.tables(dx)
    r3 = math.sqrt(3.0)
    allowed = np.array([(2 + r3) / 6, 1 / 6, (2 - r3) / 6])
    for v in Nq.ravel():
        assert np.min(np.abs(allowed - v)) < 1e-15
    # node a is closest to Gauss point q = a (same quadrant)
    assert np.allclose(np.diag(Nq), (2 + r3) / 6, rtol=0, atol=1e-15)
    assert np.allclose(Nq.sum(1), 1.0, atol=1e-15)                 # partition of unity
    assert np.allclose(dN.sum(1), 0.0, atol=1e-15)                  # gradients sum to 0
    assert abs(w.sum() - dx * dx) < 1e-12                           # weights sum to the area


def test_q1_mass_matrix_closed_form():
    """Scalar consistent mass = dx^2/36 [[4,2,1,2],[2,4,2,1],[1,2,4,2],[2,1,2,4]]."""
    dx = 2.5
    Nq, _, w = fem.tables(dx)
    Mass = np.einsum("q,qa,qb->ab", w, Nq, Nq)
    ref = dx * dx / 36 * np.array([[4, 2, 1, 2], [2, 4, 2, 1], [1, 2, 4, 2], [2, 1, 2, 4]])
    assert np.allclose(Mass, ref, rtol=1e-14, atol=0)


def test_gauss_exactness():
    """2x2 Gauss integrates xi^2 eta^2 -> 4/9 and xi -> 0 on the reference square."""
    s = sum(xi * xi * eta * eta for xi, eta in fem.QPTS)
    assert abs(s - 4 / 9) < 1e-15
    assert abs(sum(xi for xi, _ in fem.QPTS)) < 1e-15


def test_q1_stiffness_closed_form():
    """Laplacian element stiffness of Q1 on a square: diag 2/3, edge -1/6, opposite -1/3."""
    Nq, dN, w = fem.tables(7.0)
    K = np.einsum("q,qam,qbm->ab", w, dN, dN)
    ref = np.array([[4, -1, -2, -1], [-1, 4, -1, -2], [-2, -1, 4, -1], [-1, -2, -1, 4]]) / 6
    assert np.allclose(K, ref, atol=1e-14)


# ------------------------------------------------------------- pointwise rheology
def test_delta_two_ways():
    """eq:Delta == tau-form == Hibler's expansion; Delta^2 - 2 tau:tau = Dmin^2."""
    rng = np.random.default_rng(1)
    G = rng.standard_normal((1000, 2, 2)) * 1e-6
    eps = M.strain_rate(G)
    e, dmin = 2.0, 2e-9
    d1 = M.delta_hibler(eps, e, dmin)
    tau = M.tau_of(eps, e)
    d2 = M.delta_tau(tau, dmin)
    e11, e22, e12 = eps[:, 0, 0], eps[:, 1, 1], eps[:, 0, 1]
    d3 = np.sqrt((e11 ** 2 + e22 ** 2) * (1 + e ** -2) + 4 * e ** -2 * e12 ** 2
                 + 2 * e11 * e22 * (1 - e ** -2) + dmin ** 2)
    assert np.max(np.abs(d1 - d2) / d1) < 1e-14
    assert np.max(np.abs(d1 - d3) / d1) < 1e-14
    assert np.allclose(d2 ** 2 - 2 * M.frob(tau, tau), dmin ** 2, rtol=1e-6, atol=0)


def test_tau_examples():
    """SPEC-style hand examples: eps = I -> tau = I; eps = diag(1,-1), e=2 -> tau = diag(.5,-.5)."""
    assert np.allclose(M.tau_of(np.eye(2), 2.0), np.eye(2))
    assert np.allclose(M.tau_of(np.diag([1.0, -1.0]), 2.0), np.diag([0.5, -0.5]))
    assert np.allclose(M.strain_rate(np.array([[0.0, 1.0], [0.0, 0.0]])), [[0, 0.5], [0.5, 0]])


def test_sigma_pairing():
    """sigma:grad phi == (P/Delta) tau(v):tau(phi) - (P/2) tr eps(phi) (eq:sigma)."""
    rng = np.random.default_rng(2)
    Gv = rng.standard_normal((500, 2, 2)) * 1e-6
    Gp = rng.standard_normal((500, 2, 2))
    P = rng.uniform(1e3, 1e4, 500)
    e, dmin = 2.0, 2e-9
    sig = M.sigma_hibler(M.strain_rate(Gv), P, e, dmin)
    lhs = M.frob(sig, Gp)
    tv = M.tau_of(M.strain_rate(Gv), e)
    tp = M.tau_of(M.strain_rate(Gp), e)
    D = M.delta_tau(tv, dmin)
    rhs = P / D * M.frob(tv, tp) - P / 2 * M.trace(M.strain_rate(Gp))
    scale = np.abs(P / D * np.abs(tv).sum((1, 2)) * np.abs(tp).sum((1, 2))) + P
    assert np.max(np.abs(lhs - rhs) / scale) < 1e-14


def test_yield_curve_equivalence():
    """sqrt(2 pi:pi) for pi = tau/Delta (eq:pi) equals the elliptical yield
    measure ((sI + P/2)/(P/2))^2 + (sII/(P/(2e)))^2 of the Hibler stress, and is < 1."""
    rng = np.random.default_rng(3)
    G = rng.standard_normal((500, 2, 2)) * 10.0 ** rng.uniform(-12, -5, (500, 1, 1))
    e, dmin, P = 2.0, 2e-9, 5000.0
    eps = M.strain_rate(G)
    tau = M.tau_of(eps, e)
    D = M.delta_tau(tau, dmin)
    pi = tau / D[:, None, None]
    m_pi = 2 * M.frob(pi, pi)
    sig = M.sigma_hibler(eps, np.full(500, P), e, dmin)
    sI = 0.5 * M.trace(sig)
    dev = M.deviator(sig)
    sII = np.sqrt(0.5 * M.frob(dev, dev))
    ell = ((sI + P / 2) / (P / 2)) ** 2 + (sII / (P / (2 * e))) ** 2
    assert np.allclose(m_pi, ell, rtol=1e-9, atol=1e-14)
    assert np.all(m_pi < 1.0)


def test_ice_strength_and_forcing():
    """P = P* H exp(-C(1-A)); drag laws: homogeneity, hand values."""
    assert M.ice_strength(np.array([1.0]), np.array([1.0]), PRM)[0] == PRM.P_star
    assert np.isclose(M.ice_strength(np.array([2.0]), np.array([0.5]), PRM)[0], 2 * 27500 * math.exp(-10))
    va = np.array([[5.0, 5.0]])
    assert np.allclose(M.tau_atm(va, PRM), 1.2e-3 * 1.3 * math.sqrt(50) * va)
    assert np.allclose(M.tau_atm(2 * va, PRM), 4 * M.tau_atm(va, PRM))
    p1 = dataclasses.replace(PRM, C_o=1.0, rho_o=1.0)
    # v = 0, v_o = (1,0): drag = (1,0), -tau_ocean' = [[2,0],[0,1]]
    assert np.allclose(M.tau_ocean(np.zeros((1, 2)), np.array([[1.0, 0.0]]), p1), [[1.0, 0.0]])
    assert np.allclose(M.ocean_drag_coeff(np.zeros((1, 2)), np.array([[1.0, 0.0]]), p1), [[[2, 0], [0, 1]]])
    # central FD of tau_ocean w.r.t. v
    rng = np.random.default_rng(4)
    v, vo = rng.standard_normal((1, 2)), rng.standard_normal((1, 2))
    D = M.ocean_drag_coeff(v, vo, PRM)[0]
    h = 1e-6
    for m in range(2):
        dv = np.zeros((1, 2)); dv[0, m] = h
        fd = (M.tau_ocean(v + dv, vo, PRM) - M.tau_ocean(v - dv, vo, PRM))[0] / (2 * h)
        assert np.allclose(-fd, D[:, m], rtol=1e-7)


def test_sv_coefficient_self_adjoint_and_spd():
    """eq:modification makes C self-adjoint; it stays positive definite for ANY pi:
    lambda_min(C) >= (P/Delta)(1 - sqrt2 |tau|/Delta) > 0 (derivation in SURVEY §8(c)-4)."""
    rng = np.random.default_rng(5)
    e, dmin = 2.0, 2e-9
    basis = [np.array([[1.0, 0], [0, 0]]), np.array([[0, 1.0], [1.0, 0]]) / math.sqrt(2), np.array([[0, 0], [0, 1.0]])]
    worst = np.inf
    for _ in range(2000):
        tau = M.strain_rate(rng.standard_normal((2, 2))) * 10.0 ** rng.uniform(-11, -6)
        pi = M.strain_rate(rng.standard_normal((2, 2))) * rng.uniform(0, 3)
        D = M.delta_tau(tau, dmin)
        P = 5000.0
        Cm = np.array([[M.frob(M.coeff_apply("sv", X, tau, pi, D, P), Y) for X in basis] for Y in basis])
        assert np.allclose(Cm, Cm.T, rtol=1e-12, atol=1e-12 * abs(Cm).max())
        lmin = np.linalg.eigvalsh(0.5 * (Cm + Cm.T)).min()
        bound = P / D * (1 - math.sqrt(2 * M.frob(tau, tau)) / D)
        assert bound > 0
        worst = min(worst, lmin / bound)
    assert worst >= 1.0 - 1e-9


# ---------------------------------------------------------------- weak forms
def test_residual_vanishes_trivial():
    """P* = 0, v = v^n = 0, v_a = v_o = 0 -> R = 0 exactly (every term of eq:A/eq:F vanishes)."""
    p0 = dataclasses.replace(PRM, P_star=0.0)
    cfg, inp = wl.custom_inputs(6)
    inp.v_air[:] = 0.0
    inp.v_ocean[:] = 0.0
    pb = M.Problem(inp, p0)
    assert np.all(pb.residual(np.zeros(pb.N)) == 0.0)


def test_worked_example_2x2():
    """Golden: SURVEY §8(c)-4 worked example (hand derivation from P:397-404)."""
    g = json.load(open(os.path.join(GOLDEN, "worked_example_2x2.json")))
    n, dx = g["n"], g["dx"]
    L = n * dx
    Nn = (n + 1) ** 2
    ta = np.array(g["tau_atm"])
    speed = math.sqrt(np.linalg.norm(ta) / (PRM.C_a * PRM.rho_a))
    va = speed * ta / np.linalg.norm(ta)
    inp = wl.StepInputs(n=n, dt=g["dt"], t_new=g["dt"], h=np.full(n * n, g["h"]), A=np.ones(n * n),
                        v_prev=np.zeros(2 * Nn), v_air=np.tile(va, Nn), v_ocean=np.zeros(2 * Nn), L=L)
    pb = M.Problem(inp, PRM)
    v0 = np.zeros(pb.N)
    J = pb.jacobian(v0, np.zeros((3, 4, n * n)), "sv").toarray()
    R = pb.residual(v0)
    c = 4  # centre node of the 3x3 node grid
    P = PRM.P_star * g["h"]
    Jcc = 4 * PRM.rho_i * g["h"] * dx * dx / 9 + g["dt"] * P / PRM.delta_min * (2 / 3) * (1 + 2 / PRM.e ** 2)
    assert np.allclose(J[2 * c:2 * c + 2, 2 * c:2 * c + 2], Jcc * np.eye(2), rtol=1e-13, atol=1e-13 * Jcc)
    assert np.allclose(R[2 * c:2 * c + 2], g["dt"] * ta * dx * dx, rtol=1e-12)
    vt = np.linalg.solve(J, R)
    assert np.allclose(vt[2 * c:2 * c + 2], g["dt"] * ta * dx * dx / Jcc, rtol=1e-12)
    assert np.allclose(vt[2 * c:2 * c + 2], g["expected_vt_c"], rtol=g["expected_rel_tol"])


def _smooth_state(pb, seed=0, amp=0.05):
    """v with strain rates >> Delta_min so that central differences are meaningful."""
    return wl.random_velocity(pb.n, seed, amp=amp)


def test_energy_derivative_is_minus_residual():
    """Phi'(v)(phi) = A(v,phi) - F(phi) = -R.phi (Theorem 1 proof; reading G7)."""
    prm = dataclasses.replace(PRM, delta_min=2e-7)
    pb, _ = small_problem(8, prm=prm)
    v = _smooth_state(pb)
    rng = np.random.default_rng(7)
    d = wl.random_interior_vector(8, 8) * 0.01
    R = pb.residual(v)
    best = np.inf
    for h in (1e-2, 3e-3, 1e-3, 3e-4):
        fd = (pb.energy(v + h * d) - pb.energy(v - h * d)) / (2 * h)
        best = min(best, abs(fd + R @ d) / abs(R @ d))
    assert best < 1e-6


def test_energy_convex_midpoint():
    """Theorem 1: Phi((u+w)/2) <= (Phi(u)+Phi(w))/2; Delta - tr eps >= 0."""
    pb, _ = small_problem(8)
    rng = np.random.default_rng(8)
    for s in range(20):
        u = wl.random_velocity(8, 100 + s, amp=rng.uniform(0.01, 1))
        w = wl.random_velocity(8, 200 + s, amp=rng.uniform(0.01, 1))
        assert pb.energy(0.5 * (u + w)) <= 0.5 * (pb.energy(u) + pb.energy(w)) + 1e-9 * abs(pb.energy(u))
    _, eps, tau, D = pb.kinematics(u, pb.cells_all())
    assert np.all(D - M.trace(eps) >= 0)


def test_delta_energy_matches_direct_difference():
    """Difference-form DeltaPhi (reading G12) equals Phi(v + a vt) - Phi(v) where the direct
    difference has no cancellation (large steps), for every alpha of the backtracking."""
    pb, _ = small_problem(8)
    v = wl.random_velocity(8, 1, amp=0.02)
    vt = wl.random_velocity(8, 2, amp=0.5)
    for a in (1.0, 0.5, 0.25, 0.125):
        direct = pb.energy(v + a * vt) - pb.energy(v)
        diff = pb.delta_energy(v, vt, a)
        assert abs(direct - diff) <= 1e-9 * abs(direct)


def test_delta_energy_small_step_precision():
    """At tiny steps the direct Phi difference is roundoff, the difference form is not:
    DeltaPhi(a) / a -> Phi'(v)(vt) = -R.vt as a -> 0."""
    pb, _ = small_problem(8)
    v = wl.random_velocity(8, 1, amp=0.02)
    vt = wl.random_interior_vector(8, 3) * 1e-3
    slope = -(pb.residual(v) @ vt)
    for a in (1e-6, 1e-8):
        est = pb.delta_energy(v, vt, a) / a
        assert abs(est - slope) <= 1e-4 * abs(slope)


@pytest.mark.parametrize("kind", ["std"])
def test_jacobian_std_is_fd_of_residual(kind):
    """J_std (eq:standardNewton) = -dR/dv by central differences, <= 1e-6 rel (BASELINE.json)."""
    prm = dataclasses.replace(PRM, delta_min=2e-7)
    pb, _ = small_problem(8, prm=prm)
    v = _smooth_state(pb)
    J = pb.jacobian(v, None, kind)
    for seed in range(3):
        d = wl.random_interior_vector(8, 30 + seed)
        Jd = J @ d
        best = np.inf
        for h in (1e-3, 1e-4, 1e-5, 1e-6):
            fd = (pb.residual(v - h * d) - pb.residual(v + h * d)) / (2 * h)
            best = min(best, np.linalg.norm(Jd - fd) / np.linalg.norm(Jd))
        assert best < 1e-6


def test_jacobian_drag_term_fd():
    """The ocean-drag part of J alone is -d(drag residual)/dv: check with Delta_min huge
    (stress linear) so FD of R isolates mass + viscous + drag terms; compare J_picard == J_std there."""
    prm = dataclasses.replace(PRM, delta_min=1.0)
    pb, _ = small_problem(6, prm=prm)
    v = wl.random_velocity(6, 3, amp=2.0)
    J = pb.jacobian(v, None, "std")
    d = wl.random_interior_vector(6, 9)
    h = 1e-5
    fd = (pb.residual(v - h * d) - pb.residual(v + h * d)) / (2 * h)
    assert np.linalg.norm(J @ d - fd) <= 1e-7 * np.linalg.norm(J @ d)


def test_jacobian_sv_equals_std_at_consistent_pi():
    """At pi = tau(v)/Delta(v) (eq:pi) the sv linearisation equals the standard one,
    entrywise to 1e-12 relative to the row scale."""
    pb, _ = small_problem(8)
    v = wl.random_velocity(8, 4, amp=0.05)
    Js = pb.jacobian(v, None, "std")
    Jv = pb.jacobian(v, pb.pi_consistent(v), "sv")
    Dm = abs(Js - Jv)
    rowmax = abs(Js).max(axis=1).toarray().ravel()
    assert np.all(Dm.max(axis=1).toarray().ravel() <= 1e-12 * rowmax)


def test_jacobian_sv_is_symmetrised_literal_operator():
    """For s = 1 (sqrt(2 pi:pi) <= 1), eq:modification replaces tau(x)pi by its symmetrisation, so
    J_sv = (K + K^T)/2 with K the literal eq:linearSVNewton operator."""
    pb, _ = small_problem(8)
    v = wl.random_velocity(8, 5, amp=0.05)
    pi = wl.random_pi(8, 6, max_norm=0.99)
    K = pb.jacobian(v, pi, "sv_unmodified")
    Jv = pb.jacobian(v, pi, "sv")
    assert abs(K - K.T).max() > 1e-6 * abs(K).max()                    # K itself is not symmetric
    assert abs(Jv - 0.5 * (K + K.T)).max() <= 1e-13 * abs(K).max()


def test_jacobian_sv_scaling_when_s_gt_1():
    """With pi scaled by c >= 1/ (sqrt2|pi|) everywhere, s = c sqrt2|pi0| so the modified term is
    invariant under pi -> c pi (eq:modification P:534-539): J_sv(c pi) == J_sv(pi) when s(pi) >= 1."""
    pb, _ = small_problem(6)
    v = wl.random_velocity(6, 5, amp=0.05)
    pi = wl.random_pi(6, 7, max_norm=1.0) + 0.0
    T = M.Problem.pi_to_tensor(pi)
    nrm = np.sqrt(2 * np.sum(T * T, axis=(-2, -1)))
    pi1 = M.Problem.pi_from_tensor(T / nrm[..., None, None] * 1.5)        # s = 1.5 everywhere
    pi2 = M.Problem.pi_from_tensor(T / nrm[..., None, None] * 4.0)        # s = 4
    J1 = pb.jacobian(v, pi1, "sv")
    J2 = pb.jacobian(v, pi2, "sv")
    assert abs(J1 - J2).max() <= 1e-12 * abs(J1).max()


def test_jacobian_spd_random_pi():
    """x^T J x > 0 on interior vectors for any pi (P:970-981 + eq:modification); J symmetric."""
    pb, _ = small_problem(10)
    v = wl.random_velocity(10, 6, amp=0.05)
    pi = wl.random_pi(10, 8, max_norm=3.0)
    J = pb.jacobian(v, pi, "sv")
    assert abs(J - J.T).max() <= 1e-14 * abs(J).max()
    Ji = J[~pb.bdof][:, ~pb.bdof].toarray()
    assert np.linalg.eigvalsh(0.5 * (Ji + Ji.T)).min() > 0


def test_rigid_body_modes_in_stress_kernel():
    """tau(a - w y, b + w x) = 0, so with mass and drag switched off the stress part of
    J (std, sv, picard) annihilates rigid-body modes on rows away from the boundary."""
    prm = dataclasses.replace(PRM, rho_i=0.0, C_o=0.0)
    pb, inp = small_problem(8, prm=prm)
    pb.P = M.ice_strength(inp.h, inp.A, PRM)
    v = wl.random_velocity(8, 7, amp=0.05)
    pi = wl.random_pi(8, 9, max_norm=2.0)
    X, Y = wl.node_coords(8)
    modes = [np.stack([np.ones_like(X), 0 * X], 1).ravel(), np.stack([0 * X, np.ones_like(X)], 1).ravel(),
             np.stack([-Y, X], 1).ravel() / 512e3]
    i = np.arange(9)
    I, Jn = np.meshgrid(i, i, indexing="xy")
    deep = np.repeat(((I >= 2) & (I <= 6) & (Jn >= 2) & (Jn <= 6)).ravel(), 2)
    for kind, p in (("std", None), ("sv", pi), ("picard", None)):
        J = pb.jacobian(v, p, kind)
        scale = abs(J).max()
        for m in modes:
            assert np.max(np.abs((J @ m)[deep])) <= 1e-13 * scale * np.abs(m).max() * 9


# ---------------------------------------------------------------- dual update
def test_pi_tilde_cases():
    """eq:tautilde: pi~ = 0 for vt = 0 at consistent pi; v = pi = 0 -> pi~ = tau(vt)/Delta_min;
    at consistent pi, pi~(vt) = D(tau/Delta)[vt] (central FD, h^2 convergence)."""
    pb, _ = small_problem(8)
    v = wl.random_velocity(8, 10, amp=0.05)
    pic = pb.pi_consistent(v)
    assert np.max(np.abs(pb.pi_tilde(v, pic, np.zeros(pb.N)))) <= 1e-15 * np.max(np.abs(pic)) + 1e-300
    vt = wl.random_velocity(8, 11, amp=0.01)
    z = np.zeros(pb.N)
    _, g = pb.at_qp(vt, pb.cells_all())
    tt = M.tau_of(M.strain_rate(g), PRM.e)
    ref = M.Problem.pi_from_tensor(tt / PRM.delta_min)
    assert np.allclose(pb.pi_tilde(z, np.zeros_like(pic), vt), ref, rtol=1e-14, atol=0)
    pt = pb.pi_tilde(v, pic, vt)
    errs = []
    for h in (1e-3, 5e-4):
        fd = (pb.pi_consistent(v + h * vt) - pb.pi_consistent(v - h * vt)) / (2 * h)
        errs.append(np.max(np.abs(fd - pt)) / np.max(np.abs(pt)))
    assert errs[1] < 1e-6 and errs[1] < errs[0]


# ---------------------------------------------------------------- solvers
def test_fgmres_textbook_cases():
    """FGMRES: A = I -> 1 iteration; exact preconditioner -> 1 iteration; solution of a
    random SPD system equals the dense Cholesky solve to 1e-10."""
    rng = np.random.default_rng(12)
    b = rng.standard_normal(50)
    x, st = krylov.fgmres(lambda x: x, b)
    assert st["iters"] == 1 and np.allclose(x, b)
    Q = rng.standard_normal((60, 60))
    A = Q @ Q.T + 60 * np.eye(60)
    b = rng.standard_normal(60)
    Ainv = np.linalg.inv(A)
    x, st = krylov.fgmres(lambda x: A @ x, b, lambda r: Ainv @ r)
    assert st["iters"] == 1
    x, st = krylov.fgmres(lambda x: A @ x, b, restart=10, rtol=1e-12, maxit=1000)
    assert np.linalg.norm(x - krylov.dense_cholesky_solve(A, b)) <= 1e-10 * np.linalg.norm(x)
    d = np.diag(A).copy()
    Ad = np.diag(d)
    x, st = krylov.fgmres(lambda x: Ad @ x, b, lambda r: r / d)
    assert st["iters"] == 1


def test_fgmres_gmres_minimal_residual_property():
    """Unrestarted GMRES minimises ||b - A x|| over the Krylov space: compare iterate k with the
    least-squares solution over span{b, Ab, ..., A^{k-1} b} computed by brute force."""
    rng = np.random.default_rng(13)
    A = rng.standard_normal((40, 40)) + 8 * np.eye(40)
    b = rng.standard_normal(40)
    for k in (3, 7, 12):
        x, st = krylov.fgmres(lambda x: A @ x, b, restart=k, rtol=0.0, maxit=k)
        Kb = np.stack([np.linalg.matrix_power(A, i) @ b for i in range(k)], 1)
        Qk, _ = np.linalg.qr(Kb)
        y, *_ = np.linalg.lstsq(A @ Qk, b, rcond=None)
        assert np.linalg.norm(b - A @ x) <= np.linalg.norm(b - A @ (Qk @ y)) * (1 + 1e-8)


def test_pcg_and_fgmres_on_jacobian_match_direct():
    pb, _ = small_problem(12)
    v = wl.random_velocity(12, 14, amp=0.05)
    J = pb.jacobian(v, pb.pi_consistent(v), "sv")
    R = pb.residual(v)
    xd = krylov.sparse_direct_solve(J, R)
    xc = krylov.dense_cholesky_solve(J, R)
    assert np.linalg.norm(xd - xc) <= 1e-10 * np.linalg.norm(xc)
    xg, st = krylov.fgmres(lambda x: J @ x, R, krylov.jacobi(J), 30, 1e-12, 20000)
    assert st["converged"] and np.linalg.norm(xg - xc) <= 1e-6 * np.linalg.norm(xc)
    xp, st = krylov.pcg(lambda x: J @ x, R, krylov.jacobi(J), 1e-12, 20000)
    assert st["converged"] and np.linalg.norm(xp - xc) <= 1e-6 * np.linalg.norm(xc)


# ---------------------------------------------------------------- Newton
def test_newton_config1_quadratic_tail_and_energy_decrease():
    """Config 1 with direct solves: converges to 1e-8 (BASELINE.json), Phi strictly decreases
    (P:355-360), alpha = 1 and quadratic convergence in the tail (modifications vanish at
    convergence), final pi inside the yield ellipse up to 1e-6."""
    inp = wl.step_inputs(wl.CONFIGS[1], 0)
    v, pi, h = newton.solve_step(inp, PRM, record_iterates=True)
    assert h["converged"]
    res = np.array(h["res"]) / h["res"][0]
    assert res[-1] <= 1e-8
    assert 8 <= h["newton_iters"] <= 20
    pb = M.Problem(inp, PRM)
    phis = [pb.energy(it[0]) for it in h["iterates"]]
    assert all(h["dphi"][k] < 0 for k in range(len(h["dphi"])))
    assert all(phis[k + 1] <= phis[k] for k in range(len(phis) - 1))
    assert all(a == 1.0 for a in h["alpha"][-3:])
    # quadratic tail: r_{l+1} <= C r_l^2 with a moderate C, and the order estimate is ~2
    r = res[-4:]
    for k in range(1, 4):
        assert r[k] <= 1e3 * r[k - 1] ** 2                       # C ~ 1e2 observed
    assert r[3] / r[2] < r[2] / r[1] < r[1] / r[0]               # contraction factor shrinks
    T = M.Problem.pi_to_tensor(pi)
    assert np.sqrt(2 * np.sum(T * T, axis=(-2, -1))).max() <= 1 + 1e-6
    pc = pb.pi_consistent(v)
    Tc = M.Problem.pi_to_tensor(pc)
    assert np.sqrt(2 * np.sum(Tc * Tc, axis=(-2, -1))).max() < 1.0


def test_newton_std_vs_sv_solution_unique():
    """The discrete step is the unique minimiser of the strictly convex Phi (G28): sv
    Newton and Picard-start/std Newton on a mild case land on the same v."""
    prm = dataclasses.replace(PRM, delta_min=2e-7)
    _, inp = wl.custom_inputs(8, seed=3)
    v1, _, h1 = newton.solve_step(inp, prm, kind="sv", rtol=1e-11)
    v2, _, h2 = newton.solve_step(inp, prm, kind="std", rtol=1e-11)
    assert h1["converged"] and h2["converged"]
    assert np.linalg.norm(v1 - v2) <= 1e-8 * np.linalg.norm(v1)


def test_newton_krylov_paths_agree():
    """Jacobi-FGMRES inner solves reach the same step result as direct solves (config 1 size)."""
    _, inp = wl.custom_inputs(12, seed=5)
    v1, _, h1 = newton.solve_step(inp, PRM, linsolve="direct", rtol=1e-9)
    v2, _, h2 = newton.solve_step(inp, PRM, linsolve="jacobi_fgmres", rtol=1e-9,
                                  krylov_rtol=1e-11, krylov_maxit=20000)
    assert abs(h1["newton_iters"] - h2["newton_iters"]) <= 1
    assert np.linalg.norm(v1 - v2) <= 1e-7 * np.linalg.norm(v1)


# ------------------------------------------------------------------ Coriolis (round-2 pins)
def test_e_r_cross_right_hand_rule():
    """e_r is the upward unit normal: e_r x e_x = e_y and e_r x e_y = -e_x
    (right-hand rule z^ x x^ = y^, z^ x y^ = -x^)."""
    assert np.array_equal(M.e_r_cross(np.array([1.0, 0.0])), np.array([0.0, 1.0]))
    assert np.array_equal(M.e_r_cross(np.array([0.0, 1.0])), np.array([-1.0, 0.0]))


def test_worked_example_2x2_coriolis_and_drag():
    """Hand derivation on the 2x2-cell mesh (single interior node c), v = 0, uniform h, A = 1,
    v^n = (a, b) on every node (so v^n != v_o), uniform v_o = (u_o, w_o) and uniform tau_atm.
    Every integrand of eq:F and of the ocean term of eq:A is then a
    constant times N_c, int N_c = dx^2 (exact under 2x2 Gauss), the pressure term cancels for
    uniform P, and the viscous term vanishes at v = 0, so
        R_c = dx^2 [rho h v^n - dt rho h f_c e_r x (v^n - v_o) + dt tau_atm + dt C_o rho_o |v_o| v_o]
    with e_r x (x, y) = (-y, x).  A sign flip of the Coriolis term (in F or in e_r x) moves R_c by
    2 dt rho h f_c dx^2 |v^n - v_o| ~ 1e-3 relative, far above the 1e-12 tolerance."""
    n, dx, h, dt = 2, 16.0e3, 0.3, 1800.0
    L = n * dx
    Nn = (n + 1) ** 2
    a, b = 0.12, -0.05
    uo, wo = -0.3, 0.2
    ta = np.array([0.2, -0.1])
    speed = math.sqrt(np.linalg.norm(ta) / (PRM.C_a * PRM.rho_a))
    va = speed * ta / np.linalg.norm(ta)
    inp = wl.StepInputs(n=n, dt=dt, t_new=dt, h=np.full(n * n, h), A=np.ones(n * n),
                        v_prev=np.tile([a, b], Nn), v_air=np.tile(va, Nn), v_ocean=np.tile([uo, wo], Nn), L=L)
    pb = M.Problem(inp, PRM)
    R = pb.residual(np.zeros(pb.N))
    rh, f = PRM.rho_i * h, PRM.f_c
    dvx, dvy = a - uo, b - wo
    cor = np.array([-dvy, dvx])                       # e_r x (v^n - v_o)
    wo_vec = np.array([uo, wo])
    expect = dx * dx * (rh * np.array([a, b]) - dt * rh * f * cor + dt * ta
                        + dt * PRM.C_o * PRM.rho_o * np.linalg.norm(wo_vec) * wo_vec)
    c = 4
    assert np.allclose(R[2 * c:2 * c + 2], expect, rtol=1e-12, atol=0.0)
    flipped = expect + 2 * dx * dx * dt * rh * f * cor
    assert np.min(np.abs(R[2 * c:2 * c + 2] - flipped)) > 1e-6 * np.max(np.abs(expect))
