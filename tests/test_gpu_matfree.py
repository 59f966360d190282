"""GPU parity of the NEXT-4 row: the matrix-free Jacobian apply y = J(v, pi) x (seaice_jv_matfree,
P:512-525 + P:534-539, JFNK discussion P:545-653) against the oracle's assembled Jacobian, and
FGMRES / the Newton step with the matrix-free operator (AMG still from the assembled J)."""
import numpy as np
import pytest

from oracle import model as M
from oracle import newton
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


@pytest.mark.parametrize("kind,n", [("sv", 37), ("std", 20), ("picard", 33), ("sv", 64)])
def test_matfree_apply_matches_oracle_jacobian(kind, n):
    """Row-relative: |y_gpu - (J_ref x)|_i <= 1e-12 (|J_ref| |x|)_i on ragged tile edges."""
    _, inp = wl.custom_inputs(n, seed=11)
    ctx = make_ctx(n, jacobian=kind)
    ctx.set_inputs(inp)
    pb = M.Problem(inp, PRM)
    v = wl.random_velocity(n, 12, amp=0.05)
    pi = wl.random_pi(n, 13)
    Jo = pb.jacobian(v, pi if kind == "sv" else None, kind)
    for seed in range(2):
        x = wl.random_interior_vector(n, seed) * 1e-2
        x[::7] += 1.0  # non-zero Dirichlet entries too (rows: identity; columns: eliminated)
        bm = np.repeat(wl.boundary_mask_nodes(n), 2)
        y = ctx.jv_matfree(v, x, pi.ravel()).cpu().numpy()
        yo = Jo @ x
        scale = abs(Jo) @ np.abs(x)
        assert np.all(np.abs(y - yo) <= 1e-12 * scale + 1e-300), np.max(np.abs(y - yo) / (scale + 1e-300))
        assert np.array_equal(y[bm], x[bm])


def test_matfree_fgmres_and_newton_match():
    """FGMRES(30)+AMG with the matrix-free operator: same iteration count (+-1) and solution as with
    the assembled stencil; a config-1 Newton step with matfree = 1 matches the oracle."""
    n = 48
    _, inp = wl.custom_inputs(n, seed=3)
    v = wl.random_velocity(n, 4, amp=0.05)
    out = {}
    for mf in (0, 1):
        ctx = make_ctx(n, matfree=mf, krylov_rtol=1e-10)
        ctx.set_inputs(inp)
        R, _ = ctx.residual(v)
        ctx.assemble_jacobian(v, None, want_csr=False)
        ctx.amg_setup()
        x, st, rc = ctx.fgmres(R)
        out[mf] = (x.cpu().numpy(), st["iters"])
    assert abs(out[0][1] - out[1][1]) <= 1
    assert np.linalg.norm(out[1][0] - out[0][0]) <= 1e-8 * np.linalg.norm(out[0][0])
    cfg = wl.CONFIGS[1]
    inp = wl.step_inputs(cfg, 0)
    vo, _, ho = newton.solve_step(inp, PRM)
    ctx = make_ctx(cfg.n, matfree=1, krylov_rtol=1e-12, krylov_maxit=1000)
    vg, st = ctx.solve_step(inp.dt, inp.t_new, inp.h, inp.A, inp.v_prev, inp.v_air, inp.v_ocean)
    assert st["converged"] == 1 and abs(st["newton_iters"] - ho["newton_iters"]) <= 1
    assert np.linalg.norm(vg.cpu().numpy() - vo) <= 1e-8 * np.linalg.norm(vo)
