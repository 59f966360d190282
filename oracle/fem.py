"""Q1 finite elements on the structured square mesh (ORACLE; test infrastructure).

PAPER.md P:719-723: structured quadrilateral mesh, Q1 velocity, Q0 (finite
volume) A and H.  P:740: Omega = (0, 512 km)^2.  The quadrature rule is not
stated in the paper; reading G3: 2x2 Gauss, physical weight dx^2/4.

Cell (i,j) has nodes, counter-clockwise, (i,j), (i+1,j), (i+1,j+1), (i,j+1)
with reference coordinates (xi_a, eta_a) = (-1,-1), (1,-1), (1,1), (-1,1).
Gauss points in the order (-g,-g), (g,-g), (g,g), (-g,g), g = 1/sqrt(3).
"""
from __future__ import annotations

import math

import numpy as np

XI = (-1.0, 1.0, 1.0, -1.0)
ETA = (-1.0, -1.0, 1.0, 1.0)
GAUSS = 1.0 / math.sqrt(3.0)
QPTS = ((-GAUSS, -GAUSS), (GAUSS, -GAUSS), (GAUSS, GAUSS), (-GAUSS, GAUSS))


def shape(a: int, xi: float, eta: float) -> float:
    """Bilinear basis N_a(xi, eta) = 1/4 (1 + xi_a xi)(1 + eta_a eta)."""
    return 0.25 * (1.0 + XI[a] * xi) * (1.0 + ETA[a] * eta)


def shape_grad(a: int, xi: float, eta: float, dx: float):
    """Physical gradient (dN_a/dx, dN_a/dy); the map x = x0 + (1+xi) dx/2 is affine."""
    return (0.25 * XI[a] * (1.0 + ETA[a] * eta) * 2.0 / dx,
            0.25 * ETA[a] * (1.0 + XI[a] * xi) * 2.0 / dx)


def tables(dx: float):
    """Nq[q,a], dN[q,a,m] (m = x,y derivative), weights w[q] (physical)."""
    Nq = np.zeros((4, 4))
    dN = np.zeros((4, 4, 2))
    for q, (xi, eta) in enumerate(QPTS):
        for a in range(4):
            Nq[q, a] = shape(a, xi, eta)
            dN[q, a, :] = shape_grad(a, xi, eta, dx)
    w = np.full(4, dx * dx / 4.0)
    return Nq, dN, w


def cell_nodes(n: int) -> np.ndarray:
    """[n*n, 4] node ids of every cell, cell id j*n+i."""
    i = np.arange(n)
    I, J = np.meshgrid(i, i, indexing="xy")
    I, J = I.ravel(), J.ravel()
    s = n + 1
    return np.stack([J * s + I, J * s + I + 1, (J + 1) * s + I + 1, (J + 1) * s + I], axis=1)


def boundary_nodes(n: int) -> np.ndarray:
    i = np.arange(n + 1)
    I, J = np.meshgrid(i, i, indexing="xy")
    return ((I == 0) | (I == n) | (J == 0) | (J == n)).ravel()


def boundary_dofs(n: int) -> np.ndarray:
    return np.repeat(boundary_nodes(n), 2)


def cells_touching(n: int, nodes) -> np.ndarray:
    """Sorted unique ids of the (up to 4) cells adjacent to each node in `nodes`."""
    s = n + 1
    out = []
    for nd in np.atleast_1d(nodes):
        j, i = divmod(int(nd), s)
        for cj in (j - 1, j):
            for ci in (i - 1, i):
                if 0 <= ci < n and 0 <= cj < n:
                    out.append(cj * n + ci)
    return np.unique(np.array(out, dtype=np.int64))
