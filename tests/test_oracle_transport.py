"""Pins of oracle/transport.py (reading G28) against facts
that do not come from the oracle itself: the trivial state, the textbook 1-D upwind update,
discrete conservation, the bilinear interpolant at face midpoints, and monotonicity of the
upwind update for a uniform (divergence-free) velocity."""
import numpy as np
import pytest

from oracle import transport as T
from paper_2204_10822_b200 import workloads as wl



def _fields(n, seed, lo=0.3, hi=0.7):
    rng = np.random.default_rng(seed)
    return rng.uniform(lo, hi, n * n), rng.uniform(0.2, 2.0, n * n)


def test_zero_velocity_leaves_fields_unchanged():
    n = 9
    A, H = _fields(n, 0)
    A1, H1 = T.transport_step(np.zeros(2 * (n + 1) ** 2), A, H, n, 1800.0, 1e3)
    assert np.array_equal(A1, A) and np.array_equal(H1, H)


def test_uniform_x_translation_is_textbook_1d_upwind():
    """v = (u, 0) everywhere (incl. the boundary): c_i <- c_i - (u dt/dx)(c_i - c_{i-1}), c_{-1} = inflow."""
    n, dx, dt, u, q_in = 12, 2.0e3, 600.0, 1.5, 0.25
    rng = np.random.default_rng(1)
    q = rng.uniform(0.0, 1.0, n * n)
    v = np.zeros(2 * (n + 1) ** 2)
    v[0::2] = u
    ux, uy = T.face_velocities(v, n)
    out = T.advect_step(q, ux, uy, dt, dx, q_in, None, None).reshape(n, n)
    Q = q.reshape(n, n)
    c = u * dt / dx
    for j in range(n):
        for i in range(n):
            left = Q[j, i - 1] if i > 0 else q_in
            assert abs(out[j, i] - (Q[j, i] - c * (Q[j, i] - left))) <= 1e-15
    # the same in y with v = (0, w), w < 0: inflow through the north boundary
    w = -0.8
    v = np.zeros(2 * (n + 1) ** 2)
    v[1::2] = w
    ux, uy = T.face_velocities(v, n)
    out = T.advect_step(q, ux, uy, dt, dx, q_in, None, None).reshape(n, n)
    c = -w * dt / dx
    for j in range(n):
        for i in range(n):
            up = Q[j + 1, i] if j + 1 < n else q_in
            assert abs(out[j, i] - (Q[j, i] - c * (Q[j, i] - up))) <= 1e-15


def test_conservation_with_no_boundary_inflow():
    n, dx, dt = 16, 1.0e3, 30.0
    A, H = _fields(n, 2)
    v = wl.random_velocity(n, 3, amp=0.2)  # zero on the boundary nodes
    ux, uy = T.face_velocities(v, n)
    assert np.max(np.abs(ux)) * dt / dx <= 1.0 and np.max(np.abs(uy)) * dt / dx <= 1.0
    for q in (A, H):
        out = T.advect_step(q, ux, uy, dt, dx, 7.0, None, None)  # inflow value never used
        assert abs(out.sum() - q.sum()) <= 1e-12 * q.sum()


def test_face_velocity_is_bilinear_interpolant_at_face_midpoint():
    n = 7
    v = wl.random_velocity(n, 4, amp=1.0)
    s = n + 1
    ux, uy = T.face_velocities(v, n)

    def q1(comp, i, j, xi, eta):  # bilinear interpolant on cell (i, j) at reference (xi, eta)
        nodes = [(i, j), (i + 1, j), (i + 1, j + 1), (i, j + 1)]
        ref = [(-1, -1), (1, -1), (1, 1), (-1, 1)]
        return sum(0.25 * (1 + a * xi) * (1 + b * eta) * v[2 * (nj * s + ni) + comp]
                   for (ni, nj), (a, b) in zip(nodes, ref))

    for j in range(n):
        for i in range(n):
            assert abs(ux[j, i] - q1(0, i, j, -1.0, 0.0)) <= 1e-14   # west face of cell (i, j)
            assert abs(ux[j, i + 1] - q1(0, i, j, 1.0, 0.0)) <= 1e-14
            assert abs(uy[j, i] - q1(1, i, j, 0.0, -1.0)) <= 1e-14
            assert abs(uy[j + 1, i] - q1(1, i, j, 0.0, 1.0)) <= 1e-14


def test_uniform_diagonal_velocity_is_monotone_and_clamps():
    n, dx, dt = 10, 1.0e3, 200.0
    rng = np.random.default_rng(5)
    q = rng.uniform(0.1, 0.9, n * n)
    v = np.zeros(2 * (n + 1) ** 2)
    v[0::2], v[1::2] = 2.0, 1.5  # CFL (2 + 1.5) * 0.2 = 0.7
    ux, uy = T.face_velocities(v, n)
    out = T.advect_step(q, ux, uy, dt, dx, 0.5, None, None)
    assert out.min() >= min(q.min(), 0.5) - 1e-15 and out.max() <= max(q.max(), 0.5) + 1e-15
    # clamping: A to [0, 1], H to [0, inf)
    A = np.full(n * n, 0.99)
    A[5] = 0.0
    v = wl.random_velocity(n, 6, amp=5.0)
    A1, H1 = T.transport_step(v, A, np.full(n * n, 1e-3), n, 600.0, 1.0e3)
    assert A1.min() >= 0.0 and A1.max() <= 1.0 and H1.min() >= 0.0


def test_cfl_number_closed_form_and_subcycling():
    """Uniform v = (u, w), u, w > 0: every cell's outflow is u + w, so CFL = dt (u + w)/dx; with
    CFL = 2.5 the step is ceil(2.5) = 3 textbook upwind sub-steps of dt/3 (1-D check in x with
    w = 0: c <- c - (u dt/3dx)(c - c_left) three times)."""
    n, dx, u, w = 8, 1.0e3, 1.5, 1.0
    v = np.zeros(2 * (n + 1) ** 2)
    v[0::2], v[1::2] = u, w
    ux, uy = T.face_velocities(v, n)
    assert abs(T.cfl_number(ux, uy, 400.0, dx) - 400.0 * (u + w) / dx) <= 1e-15
    v[1::2] = 0.0
    dt = 2.5 * dx / u
    rng = np.random.default_rng(7)
    A = rng.uniform(0.2, 0.8, n * n)
    A1, H1, cfl, m = T.transport_step(v, A, A.copy(), n, dt, dx, A_in=0.4, H_in=0.4, info=True)
    assert m == 3 and abs(cfl - 2.5) <= 1e-15
    Q = A.reshape(n, n).copy()
    c = u * dt / 3 / dx
    for _ in range(3):
        left = np.concatenate([np.full((n, 1), 0.4), Q[:, :-1]], axis=1)
        Q = Q - c * (Q - left)
    assert np.max(np.abs(A1 - Q.ravel())) <= 1e-15 and np.max(np.abs(H1 - Q.ravel())) <= 1e-15
    assert A1.min() >= 0.2 - 1e-15 and A1.max() <= 0.8 + 1e-15   # monotone: no clamp needed
