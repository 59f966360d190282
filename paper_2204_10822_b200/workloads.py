"""Seeded synthetic workloads (BASELINE.json configs 1-5).

This module holds ONLY input generation: seeded random draws and the analytic
forcing fields named in BASELINE.json.  It contains none of the method's
arithmetic (no rheology, no quadrature, no drag law), so both the CPU oracle
(`oracle/`) and the CUDA path may import it (task rule: "only the seeded input
generators serve both").

Readings of BASELINE.json (recorded in DESIGN.md):
  G19  wind: cyclone vortex v_a = S(rho)(cos b th_hat - sin b r_hat),
       S(rho) = 15 (rho/R) exp(1 - rho/R), R = 320 km, b = 18 deg (inflow).
       Shape after PAPER.md Problem II, normalised to a 15 m/s peak.
  G20  moving centre m(t) = (256,256) km + (7/sqrt2 m/s) t (1,1), t = t_{n+1}.
  G21  ocean gyre v_o = 0.01 (-1 + 2y/L, 1 - 2x/L) m/s.
  G22  h = 0.3 + sum_{s=1..3} 0.005 sin(2 pi (x cos th_s + y sin th_s)/lam_s + phi_s)
       at cell centres (mirrors PAPER.md H_0).
  G23  numpy default_rng(seed); draw order lam(3), th(3), phi(3), then A's
       uniforms [n*n] row-major; A = 1 - U[0, 0.05].
  G24  config 5: A = 1, h_c = 2 Delta_min zeta_c / P*, zeta_c = 10^U(4,13).

Layouts: cell (i,j) -> j*n+i; node (i,j) -> j*(n+1)+i;
DOF 2*node + c (interleaved x/y).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

L_DOMAIN = 512.0e3  # m, PAPER.md P:740 / P:807


@dataclasses.dataclass(frozen=True)
class PhysParams:
    """Table 1 of PAPER.md with BASELINE.json's overrides:
    P* = 27500 N/m (G1, P:702 garbled), f_c = 1.46e-4 1/s (G2)."""
    rho_i: float = 900.0
    rho_a: float = 1.3
    rho_o: float = 1026.0
    C_a: float = 1.2e-3
    C_o: float = 5.5e-3
    P_star: float = 27500.0
    C: float = 20.0
    e: float = 2.0
    delta_min: float = 2.0e-9
    f_c: float = 1.46e-4


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    n: int
    seed: int
    steps: int
    moving: bool
    kind: str = "cyclone"  # "cyclone" | "viscosity" (config 5, G24)
    dt: float = 1800.0


CONFIGS = {
    1: Config("cfg1_tiny_32", 32, 0, 1, False),
    2: Config("cfg2_256", 256, 1, 24, True),
    3: Config("cfg3_1024", 1024, 2, 8, True),
    4: Config("cfg4_2048", 2048, 3, 4, True),
    5: Config("cfg5_4096_kernels", 4096, 4, 1, False, kind="viscosity"),
}


def sizes(n: int) -> dict:
    nn = (n + 1) ** 2
    return {"n": n, "nodes": nn, "N": 2 * nn, "cells": n * n,
            "interior_dof": 2 * (n - 1) ** 2,
            "nnz_csr": 18 * 2 * (n - 1) ** 2 + 2 * (nn - (n - 1) ** 2)}


def node_coords(n: int, L: float = L_DOMAIN):
    dx = L / n
    i = np.arange(n + 1, dtype=np.float64)
    X, Y = np.meshgrid(i * dx, i * dx, indexing="xy")  # [j, i]
    return X.ravel(), Y.ravel()


def cell_centres(n: int, L: float = L_DOMAIN):
    dx = L / n
    c = (np.arange(n, dtype=np.float64) + 0.5) * dx
    X, Y = np.meshgrid(c, c, indexing="xy")
    return X.ravel(), Y.ravel()


def cyclone_centre(t: float, moving: bool, L: float = L_DOMAIN):
    """G20."""
    m0 = 0.5 * L
    if not moving:
        return m0, m0
    d = 7.0 / math.sqrt(2.0) * t
    return m0 + d, m0 + d


def wind_nodal(n: int, t: float, moving: bool, L: float = L_DOMAIN):
    """G19: nodal air velocity [2*(n+1)^2] interleaved."""
    X, Y = node_coords(n, L)
    mx, my = cyclone_centre(t, moving, L)
    dxv, dyv = X - mx, Y - my
    rho = np.hypot(dxv, dyv)
    R = 320.0e3
    beta = math.radians(18.0)
    with np.errstate(invalid="ignore", divide="ignore"):
        rx = np.where(rho > 0, dxv / rho, 0.0)
        ry = np.where(rho > 0, dyv / rho, 0.0)
    S = 15.0 * (rho / R) * np.exp(1.0 - rho / R)
    thx, thy = -ry, rx
    ux = S * (math.cos(beta) * thx - math.sin(beta) * rx)
    uy = S * (math.cos(beta) * thy - math.sin(beta) * ry)
    out = np.empty(2 * X.size)
    out[0::2], out[1::2] = ux, uy
    return out


def ocean_nodal(n: int, L: float = L_DOMAIN):
    """G21."""
    X, Y = node_coords(n, L)
    out = np.empty(2 * X.size)
    out[0::2] = 0.01 * (-1.0 + 2.0 * Y / L)
    out[1::2] = 0.01 * (1.0 - 2.0 * X / L)
    return out


def ice_fields(cfg: Config, prm: PhysParams = PhysParams(), L: float = L_DOMAIN):
    """G22-G24: per-cell thickness h and concentration A (row-major cells)."""
    n = cfg.n
    rng = np.random.default_rng(cfg.seed)
    if cfg.kind == "viscosity":
        zeta = 10.0 ** rng.uniform(4.0, 13.0, n * n)
        A = np.ones(n * n)
        h = 2.0 * prm.delta_min * zeta / prm.P_star
        return h, A
    lam = rng.uniform(100.0e3, 500.0e3, 3)
    th = rng.uniform(0.0, math.pi, 3)
    ph = rng.uniform(0.0, 2.0 * math.pi, 3)
    Au = rng.uniform(0.0, 0.05, n * n)
    X, Y = cell_centres(n, L)
    h = np.full(n * n, 0.3)
    for s in range(3):
        h += 0.005 * np.sin(2.0 * math.pi * (X * math.cos(th[s]) + Y * math.sin(th[s])) / lam[s] + ph[s])
    return h, 1.0 - Au


@dataclasses.dataclass
class StepInputs:
    """Per-time-step inputs of the problem statement."""
    n: int
    dt: float
    t_new: float
    h: np.ndarray
    A: np.ndarray
    v_prev: np.ndarray
    v_air: np.ndarray
    v_ocean: np.ndarray
    load: np.ndarray | None = None
    L: float = L_DOMAIN


def step_inputs(cfg: Config, step: int, v_prev=None, prm: PhysParams = PhysParams(),
                h_A=None) -> StepInputs:
    """Inputs for implicit step `step` (0-based): t_{n+1} = (step+1) dt."""
    n = cfg.n
    h, A = ice_fields(cfg, prm) if h_A is None else h_A
    t_new = (step + 1) * cfg.dt
    if v_prev is None:
        v_prev = np.zeros(2 * (n + 1) ** 2)
    return StepInputs(n=n, dt=cfg.dt, t_new=t_new, h=h, A=A, v_prev=v_prev,
                      v_air=wind_nodal(n, t_new, cfg.moving), v_ocean=ocean_nodal(n))


def custom_inputs(n: int, seed: int = 0, moving: bool = False, dt: float = 1800.0):
    """Cyclone-type inputs at an arbitrary mesh size (tests)."""
    cfg = Config(f"custom_{n}", n, seed, 1, moving, dt=dt)
    return cfg, step_inputs(cfg, 0)


def problem1_inputs(n: int, L: float = L_DOMAIN, dt: float = 1800.0) -> StepInputs:
    """PAPER.md Problem I, a single momentum solve: v_o = 0, v_a = (5, 5) m/s,
    v^n = 0, H = 2A with A = 1 - 0.5 e^{-800|r|} - 0.4 e^{-90|r1|} - 0.4 e^{-90|r1 + 0.7|},
    r = 0.04 - (x/1000km - 0.25)^2 - (y/1000km - 0.25)^2, r1 = 0.1 + (2x/1000km)^2 - 2y/1000km
    (taken as printed, reading G26), evaluated at cell centres; dt = 0.5 h.  The paper uses
    f_c = 0 and a 1e4 residual reduction."""
    X, Y = cell_centres(n, L)
    xk, yk = X / 1.0e6, Y / 1.0e6
    r = 0.04 - (xk - 0.25) ** 2 - (yk - 0.25) ** 2
    r1 = 0.1 + (2.0 * xk) ** 2 - 2.0 * yk
    A = 1.0 - 0.5 * np.exp(-800.0 * np.abs(r)) - 0.4 * np.exp(-90.0 * np.abs(r1)) - 0.4 * np.exp(-90.0 * np.abs(r1 + 0.7))
    A = np.clip(A, 0.0, 1.0)
    Nn = (n + 1) ** 2
    va = np.empty(2 * Nn)
    va[0::2], va[1::2] = 5.0, 5.0
    return StepInputs(n=n, dt=dt, t_new=dt, h=2.0 * A, A=A, v_prev=np.zeros(2 * Nn), v_air=va,
                      v_ocean=np.zeros(2 * Nn), L=L)


# ----------------------------------------------------------------------------- Problem II
DAY = 86400.0


def problem2_wind_nodal(n: int, t: float, L: float = L_DOMAIN) -> np.ndarray:
    """PAPER.md Problem II atmosphere (Mehlmann 2021 benchmark) at time t [s]:
    v_a = omega(x, y) v_max(t) R(alpha) (x - m(t)), R(alpha) = [[cos, sin], [-sin, cos]],
    omega = exp(-|x - m| / 100 km) / 50, with x - m in km (reading G27: peak ~11 m/s);
    v_max = 15 m/s * (-tanh((4 - t)(4 + t)/2)) for t in [0, 4] d, tanh((12 - t)(-4 + t)/2) for
    t in [4, 8] d; alpha = 72 / 81 deg; m_x = m_y = 256 + 51.2 t km (t <= 4 d), 665.6 - 51.2 t km.
    Interleaved nodal [2 (n+1)^2]."""
    td = min(max(t / DAY, 0.0), 8.0)
    if td <= 4.0:
        vmax = -15.0 * math.tanh((4.0 - td) * (4.0 + td) / 2.0)
        alpha = math.radians(72.0)
        m = 256.0 + 51.2 * td
    else:
        vmax = 15.0 * math.tanh((12.0 - td) * (-4.0 + td) / 2.0)
        alpha = math.radians(81.0)
        m = 665.6 - 51.2 * td
    X, Y = node_coords(n, L)
    dxk, dyk = X / 1.0e3 - m, Y / 1.0e3 - m
    om = np.exp(-np.sqrt(dxk ** 2 + dyk ** 2) / 100.0) / 50.0
    ca, sa = math.cos(alpha), math.sin(alpha)
    va = np.empty(2 * (n + 1) ** 2)
    va[0::2] = om * vmax * (ca * dxk + sa * dyk)
    va[1::2] = om * vmax * (-sa * dxk + ca * dyk)
    return va


def problem2_initial(n: int, L: float = L_DOMAIN):
    """Problem II initial state: v = 0, A = 1, H = 0.3 m + 0.005 m (sin(60 x/1000 km)
    + sin(30 y/1000 km)) at cell centres.  Returns (h, A, v)."""
    X, Y = cell_centres(n, L)
    h = 0.3 + 0.005 * (np.sin(60.0 * X / 1.0e6) + np.sin(30.0 * Y / 1.0e6))
    return h, np.ones(n * n), np.zeros(2 * (n + 1) ** 2)


def boundary_mask_nodes(n: int):
    i = np.arange(n + 1)
    I, J = np.meshgrid(i, i, indexing="xy")
    return ((I == 0) | (I == n) | (J == 0) | (J == n)).ravel()


def random_interior_vector(n: int, seed: int, scale: float = 1.0):
    """N(0,1) DOF vector with zero Dirichlet entries (SpMV / Krylov inputs)."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(2 * (n + 1) ** 2) * scale
    bm = np.repeat(boundary_mask_nodes(n), 2)
    x[bm] = 0.0
    return x


def random_pi(n: int, seed: int, max_norm: float = 1.5):
    """Random dual variable pi [3][4][n*n] (pi11, pi12, pi22 at the 4 Gauss points)
    with sqrt(2 pi:pi) uniform in [0, max_norm] (exercises s > 1)."""
    rng = np.random.default_rng(seed)
    raw = rng.standard_normal((3, 4, n * n))
    fro = np.sqrt(raw[0] ** 2 + 2 * raw[1] ** 2 + raw[2] ** 2)
    target = rng.uniform(0.0, max_norm, (4, n * n)) / math.sqrt(2.0)
    return raw * (target / np.maximum(fro, 1e-300))[None]


def random_velocity(n: int, seed: int, amp: float = 0.1):
    """Smooth-plus-noise velocity with zero boundary values (parity states)."""
    rng = np.random.default_rng(seed)
    X, Y = node_coords(n)
    s = np.sin(math.pi * X / L_DOMAIN) * np.sin(math.pi * Y / L_DOMAIN)
    v = np.empty(2 * X.size)
    v[0::2] = amp * s * (1 + 0.3 * rng.standard_normal(X.size))
    v[1::2] = -amp * s * (1 + 0.3 * rng.standard_normal(X.size))
    bm = np.repeat(boundary_mask_nodes(n), 2)
    v[bm] = 0.0
    return v
