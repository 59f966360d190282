"""Parity at BASELINE.json's full sizes, in the configuration bench.py runs (default params):
sampled outputs the oracle computes one by one (Jacobian rows, residual entries, SpMV
entries, dual-variable updates) plus properties that hold at any size (V-cycle symmetry,
Galerkin identity, true FGMRES residual, energy decrease of the accepted Newton step)."""
import math

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import fem
from oracle import model as M
from paper_2204_10822_b200 import workloads as wl

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
PRM = wl.PhysParams()


def np_(t):
    return t.detach().cpu().numpy()


def sample_nodes(n, k=160, seed=0):
    rng = np.random.default_rng(seed)
    s = n + 1
    special = [0, n, s * n, s * s - 1,                     # corners (boundary)
               s + 1, 2 * s - 2, s * (n - 1) + 1,         # next to the boundary
               (n // 2) * s + n // 2, s * s // 2 + 3]      # centre
    return np.unique(np.concatenate([special, rng.integers(0, s * s, k)]))


def state_for(cfg, seed=5):
    v = wl.random_velocity(cfg.n, seed, amp=0.05)
    pi = wl.random_pi(cfg.n, seed + 1, max_norm=1.5)
    return v, pi


def check_rows(ctx, pb, v, pi, nodes, kind="sv"):
    rp, ci, val = ctx.assemble_jacobian(v, pi.ravel())
    rows = np.sort(np.concatenate([2 * nodes, 2 * nodes + 1]))
    rp_h = np_(rp)
    ref = pb.jacobian_rows(v, pi, kind, nodes)
    worst = 0.0
    for r in rows:
        a, b = int(rp_h[r]), int(rp_h[r + 1])
        cols = np_(ci[a:b])
        vals = np_(val[a:b])
        g = {int(c): float(x) for c, x in zip(cols, vals)}
        o = ref[int(r)]
        scale = max(abs(x) for x in o.values())
        for c in set(g) | set(o):
            worst = max(worst, abs(g.get(c, 0.0) - o.get(c, 0.0)) / scale)
    return worst


@pytest.mark.parametrize("cfg_id", [4, 5])
def test_fullsize_jacobian_residual_spmv_sampled(cfg_id):
    cfg = wl.CONFIGS[cfg_id]
    from paper_2204_10822_b200.seaice import SeaIce
    inp = wl.step_inputs(cfg, 0)
    inp.v_prev = wl.random_velocity(cfg.n, 77, amp=0.02)
    ctx = SeaIce(cfg.n)
    ctx.set_inputs(inp)
    pb = M.Problem(inp, PRM)
    v, pi = state_for(cfg)
    nodes = sample_nodes(cfg.n)
    assert check_rows(ctx, pb, v, pi, nodes) <= 1e-12
    # residual entries, contribution-scaled
    R, nrm = ctx.residual(v)
    idx, Ro, So = pb.residual_rows(v, nodes)
    Rg = np_(R)[idx]
    assert np.all(np.abs(Rg - Ro) <= 1e-12 * So + 1e-300)
    # SpMV entries y_i = sum_j J_ij x_j with the oracle's rows
    ctx.assemble_jacobian(v, pi.ravel(), want_csr=False)
    x = wl.random_interior_vector(cfg.n, 9) * 1e-3
    y = np_(ctx.spmv(x))
    rows = pb.jacobian_rows(v, pi, "sv", nodes)
    for r, row in rows.items():
        ref = sum(val * x[c] for c, val in row.items())
        scale = sum(abs(val * x[c]) for c, val in row.items()) + 1e-300
        assert abs(y[r] - ref) <= 1e-12 * scale


def test_fullsize_pi_update_and_energy_cfg4():
    """Dual update on sampled cells and Delta Phi over the full config-4 mesh."""
    cfg = wl.CONFIGS[4]
    from paper_2204_10822_b200.seaice import SeaIce
    inp = wl.step_inputs(cfg, 0)
    inp.v_prev = wl.random_velocity(cfg.n, 78, amp=0.02)
    ctx = SeaIce(cfg.n)
    ctx.set_inputs(inp)
    pb = M.Problem(inp, PRM)
    v, pi = state_for(cfg, seed=11)
    vt = wl.random_velocity(cfg.n, 13, amp=0.01)
    pg = np_(ctx.pi_tilde(v, pi.ravel(), vt)).reshape(3, 4, -1)
    po = pb.pi_tilde(v, pi, vt)
    cells = np.random.default_rng(3).integers(0, cfg.n * cfg.n, 500)
    scale = np.abs(pi).max() + np.abs(po).max()
    assert np.max(np.abs(pg[:, :, cells] - po[:, :, cells])) <= 1e-12 * scale
    for a in (1.0, 0.25, 2.0 ** -10):
        dg = ctx.delta_energy(v, vt, [a])[0]
        do, S = pb.delta_energy(v, vt, a, with_abs=True)
        assert abs(dg - do) <= 1e-10 * abs(do) + 1e-12 * S


def test_fullsize_solver_properties_cfg4():
    """At config 4 in the bench configuration: V-cycle symmetric, Galerkin identity on level 1 -> 2,
    FGMRES true residual <= 1e-8 ||b||, accepted Newton step decreases Phi."""
    cfg = wl.CONFIGS[4]
    from paper_2204_10822_b200.seaice import SeaIce
    from test_gpu_amg import bsr_to_scipy, rows_close
    h, A = wl.ice_fields(cfg)
    va = wl.wind_nodal(cfg.n, cfg.dt, cfg.moving)
    vo = wl.ocean_nodal(cfg.n)
    ctx = SeaIce(cfg.n)
    v = torch.zeros(ctx.N, dtype=torch.float64, device="cuda")
    ctx.set_step(cfg.dt, cfg.dt, h, A, v, va, vo)
    for _ in range(4):                     # a nonlinear iterate (plastic zones present)
        d = ctx.newton_step(v)
        assert d["dphi"] < 0 and d["krylov"]["converged"] == 1
    ctx.assemble_jacobian(v, None, want_csr=False)
    nl, oc = ctx.amg_setup()
    assert nl >= 4 and oc < 3.0
    r1 = torch.randn(ctx.N, dtype=torch.float64, device="cuda")
    r2 = torch.randn(ctx.N, dtype=torch.float64, device="cuda")
    bd = wl.boundary_mask_nodes(cfg.n).repeat(2)
    r1[torch.from_numpy(bd).cuda()] = 0
    r2[torch.from_numpy(bd).cuda()] = 0
    z1, z2 = ctx.precond_apply(r1), ctx.precond_apply(r2)
    s12, s21 = float(z1 @ r2), float(r1 @ z2)
    assert abs(s12 - s21) <= 1e-10 * abs(s12)
    A1, P1, _ = ctx.amg_level(1)
    A2, _, _ = ctx.amg_level(2)
    A1s, P1s, A2s = bsr_to_scipy(A1), bsr_to_scipy(P1), bsr_to_scipy(A2)
    G = (P1s.T @ A1s @ P1s).tocsr()
    G = G + sp.diags((G.diagonal() == 0).astype(float))
    assert rows_close(A2s, G, 1.0) <= 1e-12
    R, _ = ctx.residual(v)
    ctx.assemble_jacobian(v, None, want_csr=False)
    ctx.amg_setup()
    x, st, rc = ctx.fgmres(R)
    res = R - ctx.spmv(x)
    assert float(res.norm()) <= 2e-8 * float(R.norm())
