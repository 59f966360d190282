"""Manufactured-solution pin of the oracle's discretisation (BASELINE.json north_star:
"a manufactured-solution test converges at the expected rate").

v* = U (sin(pi x/L) sin(2 pi y/L), -sin(2 pi x/L) sin(pi y/L)) vanishes on the boundary.
With v^n = v_a = v_o = 0 the continuous step (eq:momen discretised in time, P:238-253;
weak form eq:A) reads  rho H v - dt div sigma(v) - dt tau_ocean(v) = g.
g is derived symbolically (sympy) from the Hibler stress, the load
(g, phi) is integrated with 6x6 Gauss, and the discrete Newton solution must converge
to v* in L2 at rate >= 1.9 (Q1 elements: 2).
"""
import math

import numpy as np
import pytest
import sympy as syp

from oracle import fem, newton
from oracle import model as M
from paper_2204_10822_b200 import workloads as wl

L = 512.0e3
U = 0.1
PRM = wl.PhysParams(delta_min=5e-7, f_c=0.0)
H0 = 0.3


def _manufactured():
    x, y = syp.symbols("x y", real=True)
    vx = U * syp.sin(syp.pi * x / L) * syp.sin(2 * syp.pi * y / L)
    vy = -U * syp.sin(2 * syp.pi * x / L) * syp.sin(syp.pi * y / L)
    e, dmin = PRM.e, PRM.delta_min
    P = PRM.P_star * H0
    exx, eyy = syp.diff(vx, x), syp.diff(vy, y)
    exy = (syp.diff(vx, y) + syp.diff(vy, x)) / 2
    tr = exx + eyy
    dxx, dyy = exx - tr / 2, eyy - tr / 2
    Delta = syp.sqrt(2 / e ** 2 * (dxx ** 2 + dyy ** 2 + 2 * exy ** 2) + tr ** 2 + dmin ** 2)
    zeta = P / (2 * Delta)
    eta = zeta / e ** 2
    sxx = 2 * eta * dxx + zeta * tr - P / 2
    syy = 2 * eta * dyy + zeta * tr - P / 2
    sxy = 2 * eta * exy
    divx = syp.diff(sxx, x) + syp.diff(sxy, y)
    divy = syp.diff(sxy, x) + syp.diff(syy, y)
    rhoH = PRM.rho_i * H0
    speed = syp.sqrt(vx ** 2 + vy ** 2)
    co = PRM.C_o * PRM.rho_o
    dt = 1800.0
    # tau_ocean(v) with v_o = 0: co |v| (-v)
    gx = rhoH * vx - dt * divx + dt * co * speed * vx
    gy = rhoH * vy - dt * divy + dt * co * speed * vy
    f = syp.lambdify((x, y), [gx, gy, vx, vy], "numpy")
    return f


def _gauss6():
    pts, wts = np.polynomial.legendre.leggauss(6)
    return pts, wts


def _solve(n, f):
    dx = L / n
    Nn = (n + 1) ** 2
    inp = wl.StepInputs(n=n, dt=1800.0, t_new=1800.0, h=np.full(n * n, H0), A=np.ones(n * n),
                        v_prev=np.zeros(2 * Nn), v_air=np.zeros(2 * Nn), v_ocean=np.zeros(2 * Nn), L=L)
    pts, wts = _gauss6()
    cn = fem.cell_nodes(n)
    ci = np.arange(n * n) % n
    cj = np.arange(n * n) // n
    load = np.zeros(2 * Nn)
    quad = []
    for a_, (xi, wx) in enumerate(zip(pts, wts)):
        for b_, (eta, wy) in enumerate(zip(pts, wts)):
            X = (ci + 0.5 * (1 + xi)) * dx
            Y = (cj + 0.5 * (1 + eta)) * dx
            gx, gy, _, _ = f(X, Y)
            w = wx * wy * dx * dx / 4
            for a in range(4):
                Na = fem.shape(a, xi, eta)
                np.add.at(load, 2 * cn[:, a], w * Na * gx)
                np.add.at(load, 2 * cn[:, a] + 1, w * Na * gy)
            quad.append((xi, eta, w, X, Y))
    inp.load = load
    v, pi, h = newton.solve_step(inp, PRM, rtol=1e-10)
    assert h["converged"]
    err2 = 0.0
    V = v.reshape(-1, 2)
    for xi, eta, w, X, Y in quad:
        _, _, vx, vy = f(X, Y)
        vh = sum(fem.shape(a, xi, eta) * V[cn[:, a]] for a in range(4))
        err2 += np.sum(w * ((vh[:, 0] - vx) ** 2 + (vh[:, 1] - vy) ** 2))
    return math.sqrt(err2), h["newton_iters"]


def test_manufactured_solution_rate():
    f = _manufactured()
    errs = [_solve(n, f)[0] for n in (16, 32, 64)]
    rates = [math.log2(errs[k] / errs[k + 1]) for k in range(2)]
    assert rates[-1] >= 1.9, (errs, rates)
    assert errs[-1] < 2e-3 * U * L  # sanity: relative L2 error small
