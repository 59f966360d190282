"""GPU parity of the NEXT-3 row: the explicit upwind transport kernel (seaice_transport) against
oracle/transport.py, and a short Problem II time loop (transport of A, H with v^n,
then the implicit sv-Newton momentum step at t_{n+1}) against the oracle loop."""
import numpy as np
import pytest

from oracle import newton
from oracle import transport as T
from paper_2204_10822_b200 import workloads as wl

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def make_ctx(n, **kw):
    from paper_2204_10822_b200.seaice import SeaIce
    # exact-Newton comparisons against the direct-solve oracle use the fixed Krylov tolerance
    # (reading G13); the Eisenstat-Walker product default (G29) is compared with the oracle's
    # same rule where a test asks for krylov_forcing=1
    kw.setdefault("krylov_forcing", 0)
    kw.setdefault("amg_lag", 0)  # the oracle runs these tests compare with rebuild at every iteration
    return SeaIce(n, **kw)


@pytest.mark.parametrize("n", [2, 37, 256])
def test_transport_kernel_parity(n):
    """Random nodal velocity (boundary nodes included, so inflow faces occur), random A near the
    clamp and thin H: every cell equal to the oracle's face-by-face update to rounding."""
    rng = np.random.default_rng(n)
    dx = wl.L_DOMAIN / n
    v = rng.normal(0.0, 0.3, 2 * (n + 1) ** 2)
    A = np.clip(rng.uniform(0.8, 1.05, n * n), 0.0, 1.0)
    H = rng.uniform(0.0, 0.05, n * n)
    dt = 0.45 * dx / np.abs(v).max()
    Ao, Ho = T.transport_step(v, A, H, n, dt, dx, A_in=0.7, H_in=0.01)
    ctx = make_ctx(n)
    Ag, Hg = ctx.transport(dt, v, A, H, A_in=0.7, h_in=0.01)
    Ag, Hg = Ag.cpu().numpy(), Hg.cpu().numpy()
    assert np.max(np.abs(Ag - Ao)) <= 1e-14 and np.max(np.abs(Hg - Ho)) <= 1e-15
    assert Ag.min() >= 0.0 and Ag.max() <= 1.0 and Hg.min() >= 0.0


@pytest.mark.parametrize("n,courant", [(37, 2.6), (64, 7.3)])
def test_transport_cfl_guard_subcycles_like_oracle(n, courant):
    """CFL > 1 (0.5 km Problem II at dt = 1800 s exceeds it above 0.28 m/s): both sides
    report the same Courant number, take ceil(CFL) sub-steps and agree to rounding; the result
    stays in [0, 1] without relying on the clamp (monotone sub-steps)."""
    rng = np.random.default_rng(n)
    dx = wl.L_DOMAIN / n
    v = rng.normal(0.0, 0.3, 2 * (n + 1) ** 2)
    A = rng.uniform(0.2, 0.9, n * n)
    H = rng.uniform(0.0, 0.05, n * n)
    ux, uy = T.face_velocities(v, n)
    dt = courant / T.cfl_number(ux, uy, 1.0, dx)
    Ao, Ho, cflo, mo = T.transport_step(v, A, H, n, dt, dx, A_in=0.5, H_in=0.01, info=True)
    ctx = make_ctx(n)
    Ag, Hg, cflg, mg = ctx.transport(dt, v, A, H, A_in=0.5, h_in=0.01, info=True)
    assert mg == mo == int(np.ceil(courant - 1e-12)) and abs(cflg - cflo) <= 1e-14 * cflo
    assert np.max(np.abs(Ag.cpu().numpy() - Ao)) <= 1e-13 and np.max(np.abs(Hg.cpu().numpy() - Ho)) <= 1e-14


def test_transport_rejects_aliasing_and_negative_dt():
    from paper_2204_10822_b200.seaice import SeaIceError
    n = 8
    ctx = make_ctx(n)
    v = torch.zeros(ctx.N, dtype=torch.float64, device="cuda")
    A = torch.ones(n * n, dtype=torch.float64, device="cuda")
    H = torch.ones(n * n, dtype=torch.float64, device="cuda")
    from paper_2204_10822_b200.seaice import _ptr
    rc = ctx.L.seaice_transport(ctx.h, 1.0, _ptr(v), _ptr(A), _ptr(H), 1.0, 0.0, _ptr(A), _ptr(H), None, None)
    assert rc == -1  # SEAICE_EINVAL
    with pytest.raises(SeaIceError):
        ctx.transport(-1.0, v, A, H)


def test_problem2_loop_matches_oracle():
    """Three Problem II steps at n = 16 (32 km): the paper's settings (f_c = 0, 1e4 reduction,
    dt = 0.5 h).  A, H after each transport to rounding; v per step to 1e-8 relative L2;
    Newton counts +-1."""
    n, dt, steps = 16, 1800.0, 3
    prm = wl.PhysParams(f_c=0.0)
    dx = wl.L_DOMAIN / n
    h0, A0, v0 = wl.problem2_initial(n)
    vo = wl.ocean_nodal(n)
    ctx = make_ctx(n, f_c=0.0, newton_rtol=1e-4, krylov_rtol=1e-12)
    hg, Ag, vg = torch.as_tensor(h0, device="cuda"), torch.as_tensor(A0, device="cuda"), torch.as_tensor(v0, device="cuda")
    ho, Ao, vor = h0.copy(), A0.copy(), v0.copy()
    for k in range(steps):
        t_new = (k + 1) * dt
        va = wl.problem2_wind_nodal(n, t_new)
        Ag, hg = ctx.transport(dt, vg, Ag, hg)
        Ao, ho = T.transport_step(vor, Ao, ho, n, dt, dx)
        assert np.max(np.abs(Ag.cpu().numpy() - Ao)) <= 1e-13
        assert np.max(np.abs(hg.cpu().numpy() - ho)) <= 1e-13
        vg, st = ctx.solve_step(dt, t_new, hg, Ag, vg, va, vo)
        inp = wl.StepInputs(n=n, dt=dt, t_new=t_new, h=ho, A=Ao, v_prev=vor, v_air=va, v_ocean=vo)
        vor, _, hist = newton.solve_step(inp, prm, rtol=1e-4)
        assert st["converged"] == 1
        err = np.linalg.norm(vg.cpu().numpy() - vor) / np.linalg.norm(vor)
        assert err <= 1e-8, (k, err)
        assert abs(st["newton_iters"] - hist["newton_iters"]) <= 1, (k, st["newton_iters"], hist["newton_iters"])
