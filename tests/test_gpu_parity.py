"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on identical
seeded inputs.  Tolerances (BASELINE.json north_star):
  residual  contribution-scaled  |R_gpu - R_ref|_i <= 1e-12 S_i
  Jacobian  row-relative         max_j |J_gpu - J_ref|_ij <= 1e-12 max_j |J_ref|_ij
  v per step                     relative L2 1e-8;  Newton count +-1;  FGMRES count +-10 %
"""
import math

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import krylov, newton
from oracle import model as M
from paper_2204_10822_b200 import workloads as wl

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
PRM = wl.PhysParams()


def make_ctx(n, **kw):
    from paper_2204_10822_b200.seaice import SeaIce
    # exact-Newton comparisons against the direct-solve oracle use the fixed Krylov tolerance
    # (reading G13); the Eisenstat-Walker product default (G29) is compared with the oracle's
    # same rule where a test asks for krylov_forcing=1
    kw.setdefault("krylov_forcing", 0)
    kw.setdefault("amg_lag", 0)  # the oracle runs these tests compare with rebuild at every iteration
    return SeaIce(n, **kw)


def to_np(t):
    return t.detach().cpu().numpy()


def gpu_csr(ctx, v, pi=None):
    rp, ci, val = ctx.assemble_jacobian(v, pi)
    return sp.csr_matrix((to_np(val), to_np(ci), to_np(rp)), shape=(ctx.N, ctx.N))


def assert_rows_close(Jg, Jo, tol=1e-12):
    D = (Jg - Jo).tocsr()
    dmax = abs(D).max(axis=1).toarray().ravel()
    rmax = abs(Jo).max(axis=1).toarray().ravel()
    bad = dmax > tol * rmax
    assert not bad.any(), f"{bad.sum()} rows off; worst {np.max(dmax / np.maximum(rmax, 1e-300)):.3e}"


def state(n, seed, amp=0.05):
    return wl.random_velocity(n, seed, amp=amp)


@pytest.fixture(scope="module", params=[1])
def cfg1(request):
    cfg = wl.CONFIGS[request.param]
    inp = wl.step_inputs(cfg, 0)
    inp.v_prev = state(cfg.n, 99, amp=0.02)
    return cfg, inp


# ------------------------------------------------------------------ residual / Jacobian
@pytest.mark.parametrize("n", [2, 3, 32, 77])
def test_residual_parity(n):
    _, inp = wl.custom_inputs(n, seed=n)
    inp.v_prev = state(n, 5, amp=0.02)
    ctx = make_ctx(n)
    ctx.set_inputs(inp)
    pb = M.Problem(inp, PRM)
    for v in (np.zeros(pb.N), state(n, 1), state(n, 2, amp=1.0)):
        Rg, nrm = ctx.residual(v)
        Ro, S = pb.residual(v, with_scale=True)
        Rg = to_np(Rg)
        assert np.all(np.abs(Rg - Ro) <= 1e-12 * S + 1e-300), np.max(np.abs(Rg - Ro) / np.maximum(S, 1e-300))
        assert abs(nrm - np.linalg.norm(Ro)) <= 1e-12 * np.linalg.norm(S)


@pytest.mark.parametrize("kind", ["sv", "std", "picard"])
@pytest.mark.parametrize("n", [2, 32, 45])
def test_jacobian_parity(kind, n):
    _, inp = wl.custom_inputs(n, seed=n + 1)
    ctx = make_ctx(n, jacobian=kind)
    ctx.set_inputs(inp)
    pb = M.Problem(inp, PRM)
    v = state(n, 3)
    for pi in (pb.pi_consistent(v), wl.random_pi(n, 4, max_norm=1.5), np.zeros((3, 4, n * n))):
        Jg = gpu_csr(ctx, v, pi.ravel())
        Jo = pb.jacobian(v, pi if kind == "sv" else None, kind)
        assert_rows_close(Jg, Jo)
        # structure: 18 entries per interior row, 1 per boundary row (explicit zeros kept)
        nnz = np.diff(Jg.indptr)
        assert set(np.unique(nnz)) <= {1, 18}


@pytest.mark.parametrize("kind", ["sv", "std", "picard"])
def test_jacobian_parity_at_rest_on_drag_cutoff(kind):
    """v = v_o = 0 and pi = 0: every Gauss point sits on Delta = Delta_min and on the ocean-drag
    cut-off |w| < 1e-12 (rank-one drag term dropped, reading of S:198), the degenerate state of
    the first Newton iterate from rest; plus a state with v = v_o exactly on half the nodes."""
    n = 24
    _, inp = wl.custom_inputs(n, seed=3)
    inp.v_ocean = np.zeros_like(inp.v_ocean)
    ctx = make_ctx(n, jacobian=kind)
    ctx.set_inputs(inp)
    pb = M.Problem(inp, PRM)
    z = np.zeros(pb.N)
    Jg = gpu_csr(ctx, z, np.zeros(12 * n * n))
    Jo = pb.jacobian(z, np.zeros((3, 4, n * n)) if kind == "sv" else None, kind)
    assert_rows_close(Jg, Jo)
    Rg, _ = ctx.residual(z)
    Ro, S = pb.residual(z, with_scale=True)
    assert np.all(np.abs(to_np(Rg) - Ro) <= 1e-12 * S + 1e-300)
    # v equal to v_o (= 0) on the left half, plastic elsewhere
    v = state(n, 4)
    s = n + 1
    left = (np.arange(s * s) % s) < s // 2
    v[np.repeat(left, 2)] = 0.0
    pi = pb.pi_consistent(v)
    Jg = gpu_csr(ctx, v, pi.ravel())
    Jo = pb.jacobian(v, pi if kind == "sv" else None, kind)
    assert_rows_close(Jg, Jo)


def test_spmv_parity():
    n = 64
    _, inp = wl.custom_inputs(n, seed=7)
    ctx = make_ctx(n)
    ctx.set_inputs(inp)
    pb = M.Problem(inp, PRM)
    v = state(n, 8)
    pi = wl.random_pi(n, 9)
    Jo = pb.jacobian(v, pi, "sv")
    ctx.assemble_jacobian(v, pi.ravel(), want_csr=False)
    for seed in range(3):
        x = wl.random_interior_vector(n, seed) * 1e-3
        yg = to_np(ctx.spmv(x))
        yo = Jo @ x
        scale = abs(Jo) @ np.abs(x)
        assert np.all(np.abs(yg - yo) <= 1e-12 * scale + 1e-300)


def test_pi_init_and_pi_tilde_parity():
    n = 40
    _, inp = wl.custom_inputs(n, seed=11)
    inp.v_prev = state(n, 12, amp=0.05)
    ctx = make_ctx(n)
    ctx.set_inputs(inp)
    pb = M.Problem(inp, PRM)
    pi0 = to_np(ctx.get_pi()).reshape(3, 4, n * n)
    ref0 = pb.pi_consistent(pb.v_prev)
    assert np.max(np.abs(pi0 - ref0)) <= 1e-13
    v = state(n, 13)
    vt = state(n, 14, amp=0.01)
    for pi in (ref0, wl.random_pi(n, 15, max_norm=2.0)):
        pg = to_np(ctx.pi_tilde(v, pi.ravel(), vt)).reshape(3, 4, n * n)
        po = pb.pi_tilde(v, pi, vt)
        scale = np.abs(pi).max() + np.abs(po).max()
        assert np.max(np.abs(pg - po)) <= 1e-12 * scale


def test_delta_energy_parity():
    n = 48
    _, inp = wl.custom_inputs(n, seed=21)
    inp.v_prev = state(n, 22, amp=0.02)
    ctx = make_ctx(n)
    ctx.set_inputs(inp)
    pb = M.Problem(inp, PRM)
    v = state(n, 23, amp=0.05)
    vt = state(n, 24, amp=0.05)
    alphas = [2.0 ** -k for k in range(12)]
    dg = ctx.delta_energy(v, vt, alphas)
    for a, d in zip(alphas, dg):
        do = pb.delta_energy(v, vt, a)
        assert abs(d - do) <= 1e-11 * abs(do) + 1e-300, (a, d, do)


def test_invalid_inputs_rejected():
    from paper_2204_10822_b200.seaice import SeaIceError, EINVAL, ESTATE
    n = 8
    _, inp = wl.custom_inputs(n)
    ctx = make_ctx(n)
    with pytest.raises(SeaIceError) as e:
        ctx.residual(np.zeros(ctx.N))
    assert e.value.code == ESTATE
    bad = inp.A.copy()
    bad[3] = 1.5
    with pytest.raises(SeaIceError) as e:
        ctx.set_step(inp.dt, inp.t_new, inp.h, bad, inp.v_prev, inp.v_air, inp.v_ocean)
    assert e.value.code == EINVAL
    hneg = inp.h.copy()
    hneg[0] = -1.0
    with pytest.raises(SeaIceError):
        ctx.set_step(inp.dt, inp.t_new, hneg, inp.A, inp.v_prev, inp.v_air, inp.v_ocean)
    va = inp.v_air.copy()
    va[5] = np.nan
    with pytest.raises(SeaIceError):
        ctx.set_step(inp.dt, inp.t_new, inp.h, inp.A, inp.v_prev, va, inp.v_ocean)
    with pytest.raises(SeaIceError):
        ctx.set_step(-1.0, inp.t_new, inp.h, inp.A, inp.v_prev, inp.v_air, inp.v_ocean)
    ctx.set_inputs(inp)  # valid inputs after failures work
    ctx.residual(np.zeros(ctx.N))


# ------------------------------------------------------------------ Krylov / Newton
def test_fgmres_jacobi_parity(cfg1):
    """FGMRES(30)-Jacobi counts vs the oracle's FGMRES with the same definition (+-10 %),
    krylov_maxit 5000 so the cap does not decide the count."""
    cfg, inp = cfg1
    ctx = make_ctx(cfg.n, precond="jacobi", krylov_maxit=5000, krylov_rtol=1e-8)
    ctx.set_inputs(inp)
    pb = M.Problem(inp, PRM)
    v = pb.v_prev.copy()
    pi = pb.pi_consistent(v)
    ctx.assemble_jacobian(v, pi.ravel(), want_csr=False)
    R = pb.residual(v)
    J = pb.jacobian(v, pi, "sv")
    xg, st, rc = ctx.fgmres(R)
    xo, so = krylov.fgmres(lambda x: J @ x, R, krylov.jacobi(J), 30, 1e-8, 5000)
    assert st["converged"] and so["converged"]
    assert abs(st["iters"] - so["iters"]) <= max(1, 0.1 * so["iters"]), (st, so)
    xd = krylov.sparse_direct_solve(J, R)
    assert np.linalg.norm(to_np(xg) - xd) <= 1e-5 * np.linalg.norm(xd)


def test_newton_step_config1_parity():
    """Config 1 full implicit step: GPU Newton (Jacobi-FGMRES, tight inner tolerance) vs the
    oracle with direct solves: Newton count +-1, v to 1e-8 relative L2."""
    cfg = wl.CONFIGS[1]
    inp = wl.step_inputs(cfg, 0)
    vo, _, ho = newton.solve_step(inp, PRM)
    ctx = make_ctx(cfg.n, precond="jacobi", krylov_maxit=20000, krylov_rtol=1e-12, restart=30)
    vg, st = ctx.solve_step(inp.dt, inp.t_new, inp.h, inp.A, inp.v_prev, inp.v_air, inp.v_ocean)
    assert st["converged"] == 1
    assert abs(st["newton_iters"] - ho["newton_iters"]) <= 1, (st, ho["newton_iters"])
    vg = to_np(vg)
    assert np.linalg.norm(vg - vo) <= 1e-8 * np.linalg.norm(vo)


def test_newton_step_api_matches_solve_step():
    """seaice_newton_step loop == seaice_solve_step; determinism (bitwise) of two runs."""
    n = 24
    _, inp = wl.custom_inputs(n, seed=31)
    kw = dict(precond="jacobi", krylov_maxit=5000, krylov_rtol=1e-10)
    ctx = make_ctx(n, **kw)
    v1, st1 = ctx.solve_step(inp.dt, inp.t_new, inp.h, inp.A, inp.v_prev, inp.v_air, inp.v_ocean)
    v1b, _ = ctx.solve_step(inp.dt, inp.t_new, inp.h, inp.A, inp.v_prev, inp.v_air, inp.v_ocean)
    assert torch.equal(v1, v1b)
    ctx.set_inputs(inp)
    v = ctx.tensor(inp.v_prev).clone()
    its = 0
    for _ in range(200):
        d = ctx.newton_step(v)
        if d["converged_on_entry"]:
            break
        its += 1
        assert d["dphi"] < 0 and 0 < d["alpha"] <= 1
    assert its == st1["newton_iters"]
    assert torch.equal(v, v1)


def test_solve_step_host_buffers():
    n = 16
    _, inp = wl.custom_inputs(n, seed=41)
    ctx = make_ctx(n, precond="jacobi", krylov_maxit=5000)
    vd, st = ctx.solve_step(inp.dt, inp.t_new, inp.h, inp.A, inp.v_prev, inp.v_air, inp.v_ocean)
    T = lambda a: torch.tensor(a, dtype=torch.float64).pin_memory()
    out = torch.zeros(ctx.N, dtype=torch.float64).pin_memory()
    st2 = ctx.solve_step_host(inp.dt, inp.t_new, T(inp.h), T(inp.A), T(inp.v_prev), T(inp.v_air),
                              T(inp.v_ocean), out)
    assert torch.equal(out, vd.cpu())
    assert st2["newton_iters"] == st["newton_iters"]
