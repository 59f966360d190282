"""CPU ORACLE (test infrastructure only) — explicit transport of A and H.

The paper advances the concentration A and mean thickness H by an explicit step of
eq:model:A / eq:model:H (dA/dt + div(v A) = 0, dH/dt + div(v H) = 0) before each
implicit momentum step ("First, an explicit time step (e.g., an explicit Euler step) is
performed to compute ... A^{n+1} and H^{n+1}"), with A in [0, 1] and
A = A_in, H = H_in on the inflow boundary.  It does not state the spatial scheme;
reading G28: first-order upwind finite volumes on the Q0 cells, face-normal
velocity = average of the two Q1 nodal velocities of the face (= the Q1 interpolant at the face
midpoint), explicit Euler, then A clamped to [0, 1] and H to [0, inf).

Plain numpy, written face by face; no code shared with the CUDA path.
Pins (tests/test_oracle_transport.py): v = 0 leaves the fields unchanged; a uniform x-velocity
reproduces the textbook 1-D upwind update; total mass is conserved when no boundary face is
inflow and no clamp is active; face velocities equal the bilinear interpolant evaluated at the
face midpoint; monotonicity under CFL <= 1.
"""
from __future__ import annotations

import numpy as np


def face_velocities(v: np.ndarray, n: int):
    """Normal velocities on the (n+1) x n vertical faces (x-normal, index [j, i], face between
    cells (i-1, j) and (i, j)) and the n x (n+1) horizontal faces (y-normal, index [j, i], face
    between cells (i, j-1) and (i, j)).  v is the interleaved nodal field [2 (n+1)^2]."""
    s = n + 1
    vx = v[0::2].reshape(s, s)  # [j, i] node (i, j)
    vy = v[1::2].reshape(s, s)
    ux = np.empty((n, s))
    for j in range(n):
        for i in range(s):
            # vertical face at x = i dx spanning nodes (i, j) and (i, j+1)
            ux[j, i] = 0.5 * (vx[j, i] + vx[j + 1, i])
    uy = np.empty((s, n))
    for j in range(s):
        for i in range(n):
            # horizontal face at y = j dx spanning nodes (i, j) and (i+1, j)
            uy[j, i] = 0.5 * (vy[j, i] + vy[j, i + 1])
    return ux, uy


def advect_step(q: np.ndarray, ux: np.ndarray, uy: np.ndarray, dt: float, dx: float, q_in: float,
                lo: float | None, hi: float | None) -> np.ndarray:
    """One explicit-Euler first-order upwind step of dq/dt + div(v q) = 0 for the cell field q
    (row-major [n*n], cell (i, j) -> j n + i).  Flux through a face = u_f * (upwind value) * dx;
    an inflow boundary face uses q_in.  The result is clamped to [lo, hi] (None: no bound)."""
    n = int(round(np.sqrt(q.size)))
    Q = q.reshape(n, n)
    out = Q.copy()
    for j in range(n):
        for i in range(n):
            div = 0.0
            # west face (x = i dx): positive u flows into the cell
            u = ux[j, i]
            up = (Q[j, i - 1] if i > 0 else q_in) if u > 0.0 else Q[j, i]
            div -= u * up
            # east face (x = (i+1) dx): positive u flows out of the cell
            u = ux[j, i + 1]
            up = Q[j, i] if u > 0.0 else (Q[j, i + 1] if i + 1 < n else q_in)
            div += u * up
            # south face
            u = uy[j, i]
            up = (Q[j - 1, i] if j > 0 else q_in) if u > 0.0 else Q[j, i]
            div -= u * up
            # north face
            u = uy[j + 1, i]
            up = Q[j, i] if u > 0.0 else (Q[j + 1, i] if j + 1 < n else q_in)
            div += u * up
            out[j, i] = Q[j, i] - dt * dx * div / (dx * dx)
    if lo is not None:
        out = np.maximum(out, lo)
    if hi is not None:
        out = np.minimum(out, hi)
    return out.ravel()


def cfl_number(ux: np.ndarray, uy: np.ndarray, dt: float, dx: float) -> float:
    """max over cells of dt/dx * (sum of the cell's outflow face velocities).  The upwind update
    q' = q (1 - dt/dx out) + dt/dx sum_in u q_nb is a convex combination (monotone) iff this
    is <= 1 (the 2-D upwind CFL condition)."""
    n = ux.shape[0]
    worst = 0.0
    for j in range(n):
        for i in range(n):
            out = max(-ux[j, i], 0.0) + max(ux[j, i + 1], 0.0) + max(-uy[j, i], 0.0) + max(uy[j + 1, i], 0.0)
            worst = max(worst, dt / dx * out)
    return worst


def transport_step(v: np.ndarray, A: np.ndarray, H: np.ndarray, n: int, dt: float, dx: float,
                   A_in: float = 1.0, H_in: float = 0.0, info: bool = False):
    """A^{n+1}, H^{n+1} from (v^n, A^n, H^n): A in [0, 1], H >= 0.
    CFL guard (reading G28): if cfl_number > 1 the step is m = ceil(CFL) sub-steps of dt/m
    with the same v.  info=True also returns (cfl, m)."""
    ux, uy = face_velocities(v, n)
    cfl = cfl_number(ux, uy, dt, dx)
    m = int(np.ceil(cfl)) if cfl > 1.0 else 1
    for _ in range(m):
        A, H = (advect_step(A, ux, uy, dt / m, dx, A_in, 0.0, 1.0),
                advect_step(H, ux, uy, dt / m, dx, H_in, 0.0, None))
    return (A, H, cfl, m) if info else (A, H)
