"""The implicit VP momentum step and its stress-velocity linearisation (ORACLE).

Test infrastructure only.  Written in the paper's tensor notation: strain rates,
tau and pi are 2x2 matrices and ":" is the Frobenius product.  Every function
cites the PAPER.md passage it follows (P:<line>).

Per-quadrature-point definitions
  eps(v)  = 1/2 (grad v + grad v^T)
  tau(v)  = e^-1 eps' + 1/2 tr(eps) I
  Delta   = sqrt(Delta_min^2 + 2 tau:tau)
  P       = P* H exp(-C(1-A))
  tau_atm = C_a rho_a |v_a| v_a ; tau_ocean = C_o rho_o |v_o-v|(v_o-v)
Weak forms
  A(v,phi) = (rho H v, phi) + dt (sigma, grad phi) - dt (tau_ocean(v), phi)      eq:A
  (sigma, grad phi) = (P/Delta tau(v), tau(phi)) - (P/2, tr eps(phi))            eq:sigma P:397-404
  F(phi)   = (rho H v^n, phi) - dt (rho H f_c e_r x (v^n - v_o), phi) + dt (tau_atm, phi)  eq:F P:330-331
  R(v)     = F - A(v)   (Dirichlet entries 0)
Energy  eq:energy P:261-268.   sv Jacobian eq:linearSVNewton P:512-525 with the
modification eq:modification P:534-539; pi update eq:tautilde P:504-511 with
the same modification (confirmed by the commented derivation P:580-583).
Readings G3-G12 are listed in DESIGN.md.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp

from . import fem

EPS_DRAG = 1.0e-12  # m/s, rank-one drag derivative dropped below (reading G? / SPEC S:198)
I2 = np.eye(2)


# ----------------------------------------------------------------- pointwise
def strain_rate(G):
    """eps = 1/2 (grad v + grad v^T). G[..., k, m] = d v_k / d x_m."""
    return 0.5 * (G + np.swapaxes(G, -1, -2))


def trace(T):
    return T[..., 0, 0] + T[..., 1, 1]


def frob(A, B):
    """A : B (Frobenius product)."""
    return np.sum(A * B, axis=(-2, -1))


def deviator(eps):
    return eps - 0.5 * trace(eps)[..., None, None] * I2


def tau_of(eps, e):
    """tau = e^-1 eps' + 1/2 tr(eps) I."""
    return deviator(eps) / e + 0.5 * trace(eps)[..., None, None] * I2


def delta_tau(tau, delta_min):
    """Delta = sqrt(Delta_min^2 + 2 tau:tau)."""
    return np.sqrt(delta_min ** 2 + 2.0 * frob(tau, tau))


def delta_hibler(eps, e, delta_min):
    """eq:Delta: sqrt(2 e^-2 eps':eps' + tr(eps)^2 + Delta_min^2)."""
    d = deviator(eps)
    return np.sqrt(2.0 / e ** 2 * frob(d, d) + trace(eps) ** 2 + delta_min ** 2)


def sigma_hibler(eps, P, e, delta_min):
    """sigma = 2 eta eps' + zeta tr(eps) I - P/2 I, zeta = P/(2 Delta), eta = zeta/e^2."""
    D = delta_hibler(eps, e, delta_min)
    zeta = P / (2.0 * D)
    eta = zeta / e ** 2
    return (2.0 * eta)[..., None, None] * deviator(eps) + (zeta * trace(eps))[..., None, None] * I2 \
        - (0.5 * P)[..., None, None] * I2


def ice_strength(H, A, prm):
    """P = P* H exp(-C (1 - A))  (eq:ice-strength)."""
    return prm.P_star * H * np.exp(-prm.C * (1.0 - A))


def tau_atm(va, prm):
    """C_a rho_a |v_a| v_a  (eq:force)."""
    return prm.C_a * prm.rho_a * np.linalg.norm(va, axis=-1)[..., None] * va


def tau_ocean(v, vo, prm):
    """C_o rho_o |v_o - v| (v_o - v)  (eq:force)."""
    w = vo - v
    return prm.C_o * prm.rho_o * np.linalg.norm(w, axis=-1)[..., None] * w


def ocean_drag_coeff(v, vo, prm):
    """-tau_ocean'(v) as a 2x2 matrix: C_o rho_o (|w| I + w w^T/|w|), w = v_o - v
    (eq:standardNewton-ocean; the sign makes it the term of A').
    The rank-one part is dropped where |w| < EPS_DRAG (its limit is 0·bounded)."""
    w = vo - v
    nw = np.linalg.norm(w, axis=-1)
    D = nw[..., None, None] * I2
    safe = nw >= EPS_DRAG
    ww = np.einsum("...k,...m->...km", w, w) / np.where(safe, nw, 1.0)[..., None, None]
    D = D + np.where(safe[..., None, None], ww, 0.0)
    return prm.C_o * prm.rho_o * D


def e_r_cross(u):
    """e_r x u for the upward unit normal e_r: (-u_y, u_x)."""
    return np.stack([-u[..., 1], u[..., 0]], axis=-1)


def pi_scale(pi):
    """s = max(1, sqrt(2 pi:pi))  (eq:modification)."""
    return np.maximum(1.0, np.sqrt(2.0 * frob(pi, pi)))


def coeff_apply(kind, X, tau, pi, Delta, P):
    """The linearised stress operator C(X) for X = tau(phi_b):
      picard: (P/Delta) X
      std   : (P/Delta) X - 2P/Delta^3 (tau:X) tau              (eq:standardNewton-sigma)
      sv    : (P/Delta) X - 2P/Delta^2 M(X),
              M(X) = [(tau:X) pi + (pi:X) tau] / (2 s)           (eq:linearSVNewton + eq:modification)
    """
    base = (P / Delta)[..., None, None] * X
    if kind == "picard":
        return base
    tX = frob(tau, X)
    if kind == "std":
        return base - (2.0 * P / Delta ** 3 * tX)[..., None, None] * tau
    if kind == "sv_unmodified":
        # eq:linearSVNewton literally, before eq:modification: (2P/Delta^2)(tau (x) pi) X = (2P/Delta^2)(tau:X) pi
        return base - (2.0 * P / Delta ** 2 * tX)[..., None, None] * pi
    if kind == "sv":
        s = pi_scale(pi)
        pX = frob(pi, X)
        M = (tX / (2.0 * s))[..., None, None] * pi + (pX / (2.0 * s))[..., None, None] * tau
        return base - (2.0 * P / Delta ** 2)[..., None, None] * M
    raise ValueError(kind)


def test_tensors(dN):
    """Gradients of phi_{a,k} = N_a e_k at each qp: Gphi[q,a,k] is the 2x2 matrix
    with row k equal to grad N_a (P:207-209 applied to the test function)."""
    G = np.zeros((4, 4, 2, 2, 2))
    for q in range(4):
        for a in range(4):
            for k in range(2):
                G[q, a, k, k, :] = dN[q, a, :]
    return G


# ----------------------------------------------------------------- problem
class Problem:
    """One implicit time step: inputs (h, A, v^n, v_a, v_o, dt, t_{n+1}) -> the
    functionals of eq:t-step on the Q1 mesh."""

    def __init__(self, inp, prm):
        self.prm = prm
        self.n = n = inp.n
        self.L = float(getattr(inp, "L", 512.0e3))
        self.dx = self.L / n
        self.dt = inp.dt
        self.N = 2 * (n + 1) ** 2
        self.Nc = n * n
        self.cn = fem.cell_nodes(n)
        self.Nq, self.dN, self.w = fem.tables(self.dx)
        self.Gphi = test_tensors(self.dN)
        self.Tphi = tau_of(strain_rate(self.Gphi), prm.e)          # tau(phi_{a,k}) [q,a,k,2,2]
        self.div_phi = trace(strain_rate(self.Gphi))               # tr eps(phi_{a,k}) [q,a,k]
        self.P = ice_strength(inp.h, inp.A, prm)
        self.rhoh = prm.rho_i * inp.h
        self.v_prev = np.asarray(inp.v_prev, dtype=np.float64)
        self.v_air = np.asarray(inp.v_air, dtype=np.float64)
        self.v_ocean = np.asarray(inp.v_ocean, dtype=np.float64)
        self.load = None if inp.load is None else np.asarray(inp.load, dtype=np.float64)
        self.bdof = fem.boundary_dofs(n)

    # -- quadrature-point evaluation --------------------------------------
    def cells_all(self):
        return np.arange(self.Nc)

    def nodal_at(self, vec, cells):
        """Nodal values V[c, a, k] of a DOF vector on the given cells."""
        V = vec.reshape(-1, 2)
        return V[self.cn[cells]]

    def at_qp(self, vec, cells):
        """(values [c,q,k], gradients [c,q,k,m]) of a Q1 field at the Gauss points."""
        V = self.nodal_at(vec, cells)
        val = np.einsum("qa,cak->cqk", self.Nq, V)
        grad = np.einsum("cak,qam->cqkm", V, self.dN)
        return val, grad

    def forcing_qp(self, cells):
        va, _ = self.at_qp(self.v_air, cells)
        vo, _ = self.at_qp(self.v_ocean, cells)
        vn, _ = self.at_qp(self.v_prev, cells)
        return va, vo, vn

    def kinematics(self, v, cells):
        val, grad = self.at_qp(v, cells)
        eps = strain_rate(grad)
        tau = tau_of(eps, self.prm.e)
        Delta = delta_tau(tau, self.prm.delta_min)
        return val, eps, tau, Delta

    # -- element vectors --------------------------------------------------
    def element_F(self, cells):
        """F(phi_{a,k}) per cell (eq:F)."""
        prm, dt = self.prm, self.dt
        va, vo, vn = self.forcing_qp(cells)
        rh = self.rhoh[cells][:, None, None]
        f_q = rh * vn - dt * rh * prm.f_c * e_r_cross(vn - vo) + dt * tau_atm(va, prm)  # [c,q,k]
        Fe = np.einsum("q,cqk,qa->cak", self.w, f_q, self.Nq)
        return Fe

    def element_A(self, v, cells, with_abs=False):
        """A(v, phi_{a,k}) per cell (eq:A with eq:sigma)."""
        prm, dt = self.prm, self.dt
        val, eps, tau, Delta = self.kinematics(v, cells)
        _, vo, _ = self.forcing_qp(cells)
        P = self.P[cells][:, None]
        rh = self.rhoh[cells][:, None, None]
        mass = np.einsum("q,cqk,qa->cak", self.w, rh * val, self.Nq)
        stress_q = (P / Delta)[..., None, None] * tau                   # [c,q,2,2]
        visc = np.einsum("q,cqij,qakij->cak", self.w, stress_q, self.Tphi)
        press = np.einsum("q,cq,qak->cak", self.w, 0.5 * np.broadcast_to(P, Delta.shape), self.div_phi)
        toc = tau_ocean(val, vo, prm)                                    # [c,q,k]
        ocean = np.einsum("q,cqk,qa->cak", self.w, toc, self.Nq)
        Ae = mass + dt * (visc - press) - dt * ocean
        if not with_abs:
            return Ae
        S = (np.einsum("q,cqk,qa->cak", self.w, np.abs(rh * val), np.abs(self.Nq))
             + dt * np.abs(np.einsum("q,cqij,qakij->cqak", self.w, stress_q, self.Tphi)).sum(1)
             + dt * np.einsum("q,cq,qak->cak", self.w, 0.5 * np.abs(np.broadcast_to(P, Delta.shape)),
                              np.abs(self.div_phi))
             + dt * np.einsum("q,cqk,qa->cak", self.w, np.abs(toc), np.abs(self.Nq)))
        return Ae, S

    def scatter(self, Ee, cells):
        out = np.zeros(self.N)
        dofs = 2 * self.cn[cells][:, :, None] + np.arange(2)[None, None, :]
        np.add.at(out, dofs.ravel(), Ee.ravel())
        return out

    def F_vector(self, cells=None):
        cells = self.cells_all() if cells is None else cells
        F = self.scatter(self.element_F(cells), cells)
        if self.load is not None:
            F = F + self.load
        F[self.bdof] = 0.0
        return F

    def residual(self, v, cells=None, with_scale=False):
        """R(v) = F - A(v), Dirichlet entries 0 (reading G8/G11).
        with_scale=True also returns S_i = sum of |terms| (parity scale)."""
        cells = self.cells_all() if cells is None else cells
        if with_scale:
            Ae, Sa = self.element_A(v, cells, with_abs=True)
        else:
            Ae = self.element_A(v, cells)
        R = self.scatter(self.element_F(cells) - Ae, cells)
        if self.load is not None:
            R = R + self.load
        R[self.bdof] = 0.0
        if not with_scale:
            return R
        prm, dt = self.prm, self.dt
        va, vo, vn = self.forcing_qp(cells)
        rh = self.rhoh[cells][:, None, None]
        fabs = (np.abs(rh * vn) + dt * np.abs(rh * prm.f_c * e_r_cross(vn - vo))
                + dt * np.abs(tau_atm(va, prm)))
        Sf = np.einsum("q,cqk,qa->cak", self.w, fabs, np.abs(self.Nq))
        S = self.scatter(Sa + Sf, cells)
        if self.load is not None:
            S = S + np.abs(self.load)
        S[self.bdof] = 0.0
        return R, S

    # -- energy -------------------------------------------------------------
    def energy(self, v):
        """Phi(v) (eq:energy) with the Q1 quadrature; minus load.v if a load is set."""
        prm, dt = self.prm, self.dt
        cells = self.cells_all()
        val, eps, tau, Delta = self.kinematics(v, cells)
        va, vo, vn = self.forcing_qp(cells)
        P = self.P[:, None]
        rh = self.rhoh[:, None]
        integrand = (0.5 * rh * np.sum(val * val, -1) - rh * np.sum(vn * val, -1)
                     + dt * (0.5 * P * (Delta - trace(eps))
                             + prm.C_o * prm.rho_o / 3.0 * np.linalg.norm(vo - val, axis=-1) ** 3
                             + rh * prm.f_c * np.sum(e_r_cross(vn - vo) * val, -1)
                             - np.sum(tau_atm(va, prm) * val, -1)))
        phi = float(np.sum(integrand * self.w[None, :]))
        if self.load is not None:
            phi -= float(self.load @ v)
        return phi

    def delta_energy(self, v, vt, alpha, with_abs=False):
        """Phi(v + alpha vt) - Phi(v) in difference form (reading G12):
        the Delta and |w|^3 differences are rewritten so no O(Phi) terms cancel.
        with_abs=True also returns S = sum_q w (|t_mass| + dt(|t_plast| + |t_ocean| + |t_lin|))
        (+ |alpha load.vt|), the scale of the roundoff in the sum (reading G12b)."""
        prm, dt = self.prm, self.dt
        cells = self.cells_all()
        val0, eps0, tau0, D0 = self.kinematics(v, cells)
        dv, geps = self.at_qp(vt, cells)
        deps = strain_rate(geps)
        dtau = tau_of(deps, prm.e)
        tau1 = tau0 + alpha * dtau
        D1 = delta_tau(tau1, prm.delta_min)
        va, vo, vn = self.forcing_qp(cells)
        P = self.P[:, None]
        rh = self.rhoh[:, None]
        a = alpha
        # 1/2 rho h (|v+a vt|^2 - |v|^2) - rho h v^n.(a vt) = rho h a vt.(v - v^n) + 1/2 rho h a^2 |vt|^2,
        # with v - v^n interpolated from NODAL differences (no cancellation when v ~ v^n)
        dvn, _ = self.at_qp(v - self.v_prev, cells)
        t_mass = rh * a * np.sum(dv * dvn, -1) + 0.5 * rh * a * a * np.sum(dv * dv, -1)
        dDelta = 2.0 * a * frob(dtau, 2.0 * tau0 + a * dtau) / (D1 + D0)
        t_plast = 0.5 * P * (dDelta - a * trace(deps))
        w0 = vo - val0
        w1 = w0 - a * dv
        n0 = np.linalg.norm(w0, axis=-1)
        n1 = np.linalg.norm(w1, axis=-1)
        den = n1 + n0
        # |w1| - |w0| = (w1 - w0).(w1 + w0)/(|w1| + |w0|) with w1 - w0 = -a vt taken exactly
        # (forming w1 - w0 from w1 would lose |w0|/|a vt| digits)
        dn = np.where(den > 0, np.sum((-a * dv) * (2.0 * w0 - a * dv), -1) / np.where(den > 0, den, 1.0), 0.0)
        t_ocean = prm.C_o * prm.rho_o / 3.0 * dn * (n1 * n1 + n1 * n0 + n0 * n0)
        t_lin = a * rh * prm.f_c * np.sum(e_r_cross(vn - vo) * dv, -1) - a * np.sum(tau_atm(va, prm) * dv, -1)
        integrand = t_mass + dt * (t_plast + t_ocean + t_lin)
        d = float(np.sum(integrand * self.w[None, :]))
        S = float(np.sum((np.abs(t_mass) + dt * (np.abs(t_plast) + np.abs(t_ocean) + np.abs(t_lin))) * self.w[None, :]))
        if self.load is not None:
            lv = float(a * (self.load @ vt))
            d -= lv
            S += abs(lv)
        return (d, S) if with_abs else d

    # -- dual variable --------------------------------------------------------
    @staticmethod
    def pi_to_tensor(pi3):
        """[3][4][Nc] (pi11, pi12, pi22) -> [Nc, 4, 2, 2]."""
        p11, p12, p22 = pi3[0].T, pi3[1].T, pi3[2].T
        return np.stack([np.stack([p11, p12], -1), np.stack([p12, p22], -1)], -2)

    @staticmethod
    def pi_from_tensor(T):
        return np.stack([T[..., 0, 0].T, T[..., 0, 1].T, T[..., 1, 1].T], 0)

    def pi_consistent(self, v):
        """pi = tau(v)/Delta(v) (eq:pi); also the initial pi (reading G4)."""
        _, _, tau, D = self.kinematics(v, self.cells_all())
        return self.pi_from_tensor(tau / D[..., None, None])

    def pi_tilde(self, v, pi3, vt):
        """pi~ = -pi + tau/Delta + tau(vt)/Delta - [(tau:tau(vt)) pi + (pi:tau(vt)) tau]/(s Delta^2)
        (eq:tautilde P:504-511 with eq:modification applied)."""
        cells = self.cells_all()
        _, _, tau, D = self.kinematics(v, cells)
        _, g = self.at_qp(vt, cells)
        tt = tau_of(strain_rate(g), self.prm.e)
        pi = self.pi_to_tensor(pi3)
        s = pi_scale(pi)
        corr = (frob(tau, tt)[..., None, None] * pi + frob(pi, tt)[..., None, None] * tau) / (s * D * D)[..., None, None]
        pt = -pi + tau / D[..., None, None] + tt / D[..., None, None] - corr
        return self.pi_from_tensor(pt)

    # -- Jacobian ---------------------------------------------------------------
    def element_K(self, v, pi3, kind, cells):
        """K[c,a,k,b,m] = sum_q w [rho H N_a N_b d_km + dt C(tau(phi_bm)) : tau(phi_ak)
        + dt N_a N_b D_km]  (eq:linearSVNewton P:512-525 / eq:standardNewton P:416-433)."""
        prm, dt = self.prm, self.dt
        val, eps, tau, D = self.kinematics(v, cells)
        _, vo, _ = self.forcing_qp(cells)
        P = np.broadcast_to(self.P[cells][:, None], D.shape)
        pi = self.pi_to_tensor(pi3)[cells] if pi3 is not None else np.zeros_like(tau)
        Dr = ocean_drag_coeff(val, vo, prm)                      # [c,q,2,2]
        rh = self.rhoh[cells]
        C = len(cells)
        K = np.zeros((C, 4, 2, 4, 2))
        NN = np.einsum("qa,qb->qab", self.Nq, self.Nq)
        for b in range(4):
            for m in range(2):
                X = np.broadcast_to(self.Tphi[:, b, m], tau.shape)   # [c,q,2,2]
                CX = coeff_apply(kind, X, tau, pi, D, P)
                # viscous-plastic part for all (a,k)
                K[:, :, :, b, m] += dt * np.einsum("q,cqij,qakij->cak", self.w, CX, self.Tphi)
                for k in range(2):
                    K[:, :, k, b, m] += np.einsum("q,qa,c->ca", self.w, NN[:, :, b], rh) * (1.0 if k == m else 0.0)
                    K[:, :, k, b, m] += dt * np.einsum("q,qa,cq->ca", self.w, NN[:, :, b], Dr[:, :, k, m])
        return K

    def jacobian(self, v, pi3=None, kind="sv"):
        """Global Jacobian with symmetric Dirichlet elimination, unit diagonal
        (reading G11); scipy CSR, duplicates summed."""
        cells = self.cells_all()
        K = self.element_K(v, pi3, kind, cells)
        dofs = (2 * self.cn[:, :, None] + np.arange(2)[None, None, :]).reshape(len(cells), 8)
        rows = np.repeat(dofs, 8, axis=1).ravel()
        cols = np.tile(dofs, (1, 8)).ravel()
        J = sp.coo_matrix((K.reshape(len(cells), 64).ravel(), (rows, cols)), shape=(self.N, self.N)).tocsr()
        J.sum_duplicates()
        keep = sp.diags((~self.bdof).astype(np.float64))
        J = (keep @ J @ keep + sp.diags(self.bdof.astype(np.float64))).tocsr()
        J.eliminate_zeros()
        J.sort_indices()
        return J

    def jacobian_rows(self, v, pi3, kind, nodes):
        """Dense rows (2 per node) of the Dirichlet-eliminated Jacobian for the given
        nodes, computed from the (<=4) adjacent cells only (full-size sampling)."""
        nodes = np.atleast_1d(nodes)
        cells = fem.cells_touching(self.n, nodes)
        K = self.element_K(v, pi3, kind, cells)
        out = {}
        bnode = fem.boundary_nodes(self.n)
        for nd in nodes:
            for k in range(2):
                row = {}
                r = 2 * int(nd) + k
                if bnode[nd]:
                    out[r] = {r: 1.0}
                    continue
                for ci, c in enumerate(cells):
                    loc = np.where(self.cn[c] == nd)[0]
                    if loc.size == 0:
                        continue
                    a = int(loc[0])
                    for b in range(4):
                        nb = int(self.cn[c, b])
                        if bnode[nb]:
                            continue
                        for m in range(2):
                            col = 2 * nb + m
                            row[col] = row.get(col, 0.0) + K[ci, a, k, b, m]
                out[r] = row
        return out

    def residual_rows(self, v, nodes):
        """Residual entries (2 per node) and their scales for sampled nodes."""
        nodes = np.atleast_1d(nodes)
        cells = fem.cells_touching(self.n, nodes)
        R, S = self.residual(v, cells=cells, with_scale=True)
        idx = (2 * nodes[:, None] + np.arange(2)[None, :]).ravel()
        return idx, R[idx], S[idx]
