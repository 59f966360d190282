"""GPU AMG (setup on the GPU + V-cycle) against oracle/amg.py (same definition, independent
code) and against algebraic properties that hold at any size."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import amg as OA
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


def np_(t):
    return t.detach().cpu().numpy()


def bsr_to_scipy(d):
    v = np_(d["val"]).reshape(-1, d["br"], d["bc"])
    return sp.bsr_matrix((v, np_(d["col_idx"]), np_(d["row_ptr"])),
                         shape=(d["nbrows"] * d["br"], d["nbcols"] * d["bc"])).tocsr()


def rows_close(A, B, tol):
    D = (A - B).tocsr()
    dm = abs(D).max(axis=1).toarray().ravel()
    rm = np.maximum(abs(A).max(axis=1).toarray().ravel(), abs(B).max(axis=1).toarray().ravel())
    return np.max(dm / np.maximum(rm, 1e-300))


def newton_state(n, seed, iters):
    """An sv-Newton iterate (v_l, pi_l) of the oracle after `iters` steps (direct solves)."""
    _, inp = wl.custom_inputs(n, seed=seed)
    pb = M.Problem(inp, PRM)
    if iters == 0:
        v = pb.v_prev.copy()
        return inp, pb, v, pb.pi_consistent(v)
    _, _, h = newton.solve_step(inp, PRM, maxit=iters, rtol=0.0, record_iterates=True)
    v, pi = h["iterates"][iters]
    return inp, pb, v, pi


@pytest.mark.parametrize("nsd", [3, 4])
@pytest.mark.parametrize("n,it", [(32, 0), (32, 6), (64, 3)])
def test_hierarchy_matches_oracle(n, it, nsd):
    inp, pb, v, pi = newton_state(n, n, it)
    J = pb.jacobian(v, pi, "sv")
    H = OA.setup(J, pb, v=v, nullspace_dim=nsd)
    ctx = make_ctx(n, nullspace_dim=nsd)
    ctx.set_inputs(inp)
    ctx.assemble_jacobian(v, pi.ravel(), want_csr=False)
    nlev, oc = ctx.amg_setup()
    assert nlev == len(H["levels"])
    if nsd == 3:  # explicit zeros differ slightly; with 4 columns dropped (v = 0) columns leave
        # zero blocks the GPU stores and scipy drops, so only the level operators are compared
        assert abs(oc - H["op_complexity"]) <= 0.02 * H["op_complexity"]
    for l in range(nlev):
        A, P, agg = ctx.amg_level(l)
        Ao = H["levels"][l]["A"]
        assert rows_close(bsr_to_scipy(A), Ao, 1.0) <= 1e-11, l
        if l < nlev - 1:
            assert np.array_equal(agg, H["levels"][l]["agg"]), l
            assert rows_close(bsr_to_scipy(P), H["levels"][l]["P"], 1.0) <= 1e-11, l


def test_galerkin_and_transfer_properties():
    """Algebra of the GPU hierarchy at a size the oracle AMG would be slow at: A_c = P^T A P
    (recomputed with scipy from the GPU's own P and A), symmetry of A_c, aggregates valid."""
    n = 128
    inp, pb, v, pi = newton_state(n, 5, 0)
    ctx = make_ctx(n)
    ctx.set_inputs(inp)
    v = wl.random_velocity(n, 3, amp=0.05)
    pi = wl.random_pi(n, 4, max_norm=1.2)
    ctx.assemble_jacobian(v, pi.ravel(), want_csr=False)
    nlev, oc = ctx.amg_setup()
    assert nlev >= 2 and 1.0 < oc < 4.0
    for l in range(nlev - 1):
        A, P, agg = ctx.amg_level(l)
        Ac, _, _ = ctx.amg_level(l + 1)
        As, Ps, Acs = bsr_to_scipy(A), bsr_to_scipy(P), bsr_to_scipy(Ac)
        G = (Ps.T @ As @ Ps).tocsr()
        d = G.diagonal()
        G = G + sp.diags((d == 0).astype(float))
        assert rows_close(Acs, G, 1.0) <= 1e-12
        assert rows_close(Acs, Acs.T.tocsr(), 1.0) <= 1e-12
        assert agg.min() >= -1 and agg.max() == P["nbcols"] - 1
        assert len(np.unique(agg[agg >= 0])) == P["nbcols"]        # every aggregate non-empty


@pytest.mark.parametrize("nsd", [3, 4])
def test_vcycle_parity_and_symmetry(nsd):
    n = 48
    inp, pb, v, pi = newton_state(n, 7, 4)
    J = pb.jacobian(v, pi, "sv")
    H = OA.setup(J, pb, v=v, nullspace_dim=nsd)
    ctx = make_ctx(n, nullspace_dim=nsd)
    ctx.set_inputs(inp)
    ctx.assemble_jacobian(v, pi.ravel(), want_csr=False)
    ctx.amg_setup()
    r1 = wl.random_interior_vector(n, 1)
    r2 = wl.random_interior_vector(n, 2)
    z1 = np_(ctx.precond_apply(r1))
    z2 = np_(ctx.precond_apply(r2))
    zo = OA.vcycle(H, r1)
    assert np.linalg.norm(z1 - zo) <= 1e-9 * np.linalg.norm(zo)
    assert abs(z1 @ r2 - r1 @ z2) <= 1e-10 * abs(z1 @ r2)
    # deterministic
    assert np.array_equal(z1, np_(ctx.precond_apply(r1)))


def test_single_level_is_exact_solve():
    """N <= coarse_max_dof: the hierarchy is one dense level and M^-1 = J^-1."""
    n = 12
    inp, pb, v, pi = newton_state(n, 9, 0)
    ctx = make_ctx(n)
    ctx.set_inputs(inp)
    v = wl.random_velocity(n, 3)
    ctx.assemble_jacobian(v, pb.pi_consistent(v).ravel(), want_csr=False)
    nlev, _ = ctx.amg_setup()
    assert nlev == 1
    J = pb.jacobian(v, pb.pi_consistent(v), "sv")
    r = wl.random_interior_vector(n, 5)
    z = np_(ctx.precond_apply(r))
    assert np.linalg.norm(J @ z - r) <= 1e-10 * np.linalg.norm(r)


@pytest.mark.parametrize("nsd,method,restart", [(3, 0, 30), (4, 0, 30), (4, 0, 60), (4, 0, 12), (4, 1, 60)])
@pytest.mark.parametrize("n,it", [(32, 0), (32, 5), (64, 8)])
def test_amg_fgmres_counts_parity(n, it, nsd, method, restart):
    """AMG-FGMRES (krylov_method 0) and AMG-PCG (1) iteration counts vs the oracle's same
    definitions, with 3 or 4 near-nullspace columns (reading G30) and restart lengths 60 (the
    default, reading G13), 30 and 12 (several restarts at these sizes)."""
    inp, pb, v, pi = newton_state(n, 11, it)
    J = pb.jacobian(v, pi, "sv")
    R = pb.residual(v)
    H = OA.setup(J, pb, v=v, nullspace_dim=nsd)
    if method == 0:
        xo, so = krylov.fgmres(lambda x: J @ x, R, lambda r: OA.vcycle(H, r), restart, 1e-8, 300)
    else:
        xo, so = krylov.pcg(lambda x: J @ x, R, lambda r: OA.vcycle(H, r), 1e-8, 300)
    ctx = make_ctx(n, nullspace_dim=nsd, krylov_method=method, restart=restart)
    ctx.set_inputs(inp)
    ctx.assemble_jacobian(v, pi.ravel(), want_csr=False)
    ctx.amg_setup()
    xg, sg, rc = ctx.fgmres(R)
    assert abs(sg["iters"] - so["iters"]) <= max(1, 0.1 * so["iters"]), (sg, so)
    xd = krylov.sparse_direct_solve(J, R)
    assert np.linalg.norm(np_(xg) - xd) <= 1e-6 * np.linalg.norm(xd)


def test_multistep_parity_moving_cyclone():
    """Three consecutive implicit steps with the moving cyclone (warm starts, where the energy
    line search must resolve tiny decreases, reading G12/G12b): Newton counts +-1 and v to
    1e-8 per step vs the oracle with direct solves."""
    n = 64
    cfg = wl.Config("ms64", n, 1, 3, True)
    hA = wl.ice_fields(cfg)
    ctx = make_ctx(n, krylov_rtol=1e-10)
    vo_ = None
    vg = torch.zeros(ctx.N, dtype=torch.float64, device="cuda")
    for s in range(3):
        inp = wl.step_inputs(cfg, s, v_prev=vo_, h_A=hA)
        vo_, _, ho = newton.solve_step(inp, PRM)
        vin = vg.clone()
        vg, st = ctx.solve_step(inp.dt, inp.t_new, inp.h, inp.A, vin, inp.v_air, inp.v_ocean)
        assert st["converged"] == 1, (s, st)
        assert abs(st["newton_iters"] - ho["newton_iters"]) <= 1, (s, st["newton_iters"], ho["newton_iters"])
        assert np.linalg.norm(np_(vg) - vo_) <= 1e-8 * np.linalg.norm(vo_), s


def test_newton_amg_config1_parity():
    """Config 1 implicit step with the product path (AMG-FGMRES): Newton count +-1 and
    converged v to 1e-8 relative L2 vs the oracle with direct solves."""
    cfg = wl.CONFIGS[1]
    inp = wl.step_inputs(cfg, 0)
    vo, _, ho = newton.solve_step(inp, PRM)
    ctx = make_ctx(cfg.n, krylov_rtol=1e-10)
    vg, st = ctx.solve_step(inp.dt, inp.t_new, inp.h, inp.A, inp.v_prev, inp.v_air, inp.v_ocean)
    assert st["converged"] == 1
    assert abs(st["newton_iters"] - ho["newton_iters"]) <= 1
    assert np.linalg.norm(np_(vg) - vo) <= 1e-8 * np.linalg.norm(vo)


def test_newton_eisenstat_walker_matches_oracle():
    """Reading G29 option (krylov_forcing = 1): GPU and oracle tier B (same AMG definition, same
    forcing rule) agree on the Newton count (+-1), the per-solve FGMRES counts (+-10 % in total)
    and the converged velocity (1e-8); the forcing needs fewer Krylov iterations in total than the
    fixed 1e-8 tolerance."""
    cfg = wl.CONFIGS[1]
    inp = wl.step_inputs(cfg, 0)
    vo, _, ho = newton.solve_step(inp, PRM, linsolve="amg_fgmres", forcing=1)
    ctx = make_ctx(cfg.n, krylov_forcing=1)
    vg, st = ctx.solve_step(inp.dt, inp.t_new, inp.h, inp.A, inp.v_prev, inp.v_air, inp.v_ocean)
    assert st["converged"] == 1 and ho["converged"]
    assert abs(st["newton_iters"] - ho["newton_iters"]) <= 1
    ko = sum(k["iters"] for k in ho["krylov"])
    assert abs(st["krylov_iters_total"] - ko) <= 0.1 * ko + 2, (st["krylov_iters_total"], ko)
    assert np.linalg.norm(np_(vg) - vo) <= 1e-8 * np.linalg.norm(vo)
    ctx0 = make_ctx(cfg.n)
    _, st0 = ctx0.solve_step(inp.dt, inp.t_new, inp.h, inp.A, inp.v_prev, inp.v_air, inp.v_ocean)
    assert st["krylov_iters_total"] < st0["krylov_iters_total"]


def test_problem1_sv_converges_std_and_picard_do_not():
    """PAPER.md Problem I at 4 km: the sv Newton reaches the paper's 1e4 reduction in
    ~16 iterations while standard Newton and Picard make "little progress within 200"."""
    n = 128
    inp = wl.problem1_inputs(n)
    its = {}
    for kind in ("sv", "std", "picard"):
        ctx = make_ctx(n, f_c=0.0, newton_rtol=1e-4, newton_maxit=200, jacobian=kind)
        v, st = ctx.solve_step(inp.dt, inp.t_new, inp.h, inp.A, inp.v_prev, inp.v_air, inp.v_ocean)
        its[kind] = (st["newton_iters"], st["converged"])
    assert its["sv"][1] == 1 and its["sv"][0] <= 30
    assert its["std"][1] == 0 and its["picard"][1] == 0


@pytest.mark.parametrize("n", [37, 64, 131])
def test_fused_chebyshev_matches_per_step(n):
    """The temporally blocked finest-level Chebyshev(3) launches (cheb_fused=1: tiles; cheb_fused=2:
    y-streamed strips with the post-smoothing residual inside) perform the same arithmetic per
    node and step as one launch per step: V-cycles agree to rounding, on meshes with ragged
    edge tiles / strips and several row segments."""
    inp, pb, v, pi = newton_state(n, 3, 0)
    v = wl.random_velocity(n, 5, amp=0.05)
    pi = wl.random_pi(n, 6, max_norm=1.2)
    out = []
    for fused in (0, 1, 2):
        ctx = make_ctx(n, cheb_fused=fused)
        ctx.set_inputs(inp)
        ctx.assemble_jacobian(v, pi.ravel(), want_csr=False)
        ctx.amg_setup()
        r = wl.random_interior_vector(n, 8)
        out.append(np_(ctx.precond_apply(r)))
    for o in out[1:]:
        assert np.linalg.norm(o - out[0]) <= 1e-12 * np.linalg.norm(out[0])


@pytest.mark.parametrize("n", [48, 64, 256, 512])
def test_persistent_vcycle_tail_matches_per_launch(n):
    """vcycle_tail = 1 runs the bottom levels of the V-cycle in one cooperative launch with grid
    barriers between the phases; the operations and their order are those of the per-launch path
    (vcycle_tail = 0, the default), so V-cycles agree to rounding.  n = 48 / 64: every coarse
    level is in the tail (CTA-per-row sweeps); n = 256 / 512: the tail starts deeper and its
    first level is swept warp per row."""
    inp, pb, v, pi = newton_state(min(n, 64), 3, 0) if n <= 64 else _plastic_state(n, 21)
    if n <= 64:
        v = wl.random_velocity(n, 5, amp=0.05)
        pi = wl.random_pi(n, 6, max_norm=1.2)
    out, launches = [], []
    for tail in (0, 1):
        ctx = make_ctx(n, vcycle_tail=tail)
        ctx.set_inputs(inp)
        ctx.assemble_jacobian(v, np.asarray(pi).ravel(), want_csr=False)
        ctx.amg_setup()
        r = wl.random_interior_vector(n, 8)
        ctx.precond_apply(r)  # first application captures the V-cycle graph
        l0 = ctx.launches
        z = np_(ctx.precond_apply(r))
        launches.append(ctx.launches - l0)
        out.append(z)
        # a second right-hand side through the same captured graph (stale work vectors must not leak)
        r2 = wl.random_interior_vector(n, 9)
        out.append(np_(ctx.precond_apply(r2)))
    assert launches[1] < launches[0], launches  # the tail did replace launches
    assert np.linalg.norm(out[2] - out[0]) <= 1e-12 * np.linalg.norm(out[0])
    assert np.linalg.norm(out[3] - out[1]) <= 1e-12 * np.linalg.norm(out[1])


PATHS = ["hash1k", "hash4k", "sort_thread", "sort_group8", "sort_warp", "hash_narrow", "cta_numeric"]


def _plastic_state(n, seed):
    """A plastic linearisation point at any size without an oracle Newton run: a smooth random
    velocity (strain rates >> Delta_min everywhere) with the consistent dual variable."""
    _, inp = wl.custom_inputs(n, seed=seed)
    pb = M.Problem(inp, PRM)
    v = wl.random_velocity(n, seed + 1, amp=0.05)
    return inp, pb, v, pb.pi_consistent(v)


@pytest.mark.parametrize("n,path", [(256, 0), (512, 0), (256, 1), (256, 2), (256, 3), (256, 4), (256, 5),
                                    (256, 6)])
def test_hierarchy_matches_oracle_at_scale(n, path):
    """AMG hierarchy parity at sizes that take the SpGEMM code paths config 4 uses (verdict r1):
    same level count, identical aggregates, A_l and P_l to 1e-11 row-relative, with the automatic
    path choice (path 0) and with every product forced through each SpGEMM path (1-6); the set
    of paths config 4 (n = 2048) takes is then covered by the paths exercised here."""
    inp, pb, v, pi = _plastic_state(n, 21)
    J = pb.jacobian(v, pi, "sv")
    H = _oracle_h.get(n)
    if H is None:
        H = _oracle_h[n] = OA.setup(J, pb, v=v)
    ctx = make_ctx(n, spgemm_path=path)
    ctx.set_inputs(inp)
    ctx.assemble_jacobian(v, pi.ravel(), want_csr=False)
    nlev, oc = ctx.amg_setup()
    hits = ctx.spgemm_path_hits()
    assert nlev == len(H["levels"])
    for l in range(nlev):
        A, P, agg = ctx.amg_level(l)
        assert rows_close(bsr_to_scipy(A), H["levels"][l]["A"], 1.0) <= 1e-11, l
        if l < nlev - 1:
            assert np.array_equal(agg, H["levels"][l]["agg"]), l
            assert rows_close(bsr_to_scipy(P), H["levels"][l]["P"], 1.0) <= 1e-11, l
    _covered[(n, path)] = {PATHS[k] for k, h in enumerate(hits) if h}
    print(n, path, "levels", nlev, "spgemm paths", sorted(_covered[(n, path)]))


_covered = {}
_oracle_h = {}


def test_config4_spgemm_paths_are_parity_covered():
    """Runs after test_hierarchy_matches_oracle_at_scale (file order): the paths config 4's setup
    takes (a plastic state and a late Newton iterate of its first step) are all among those the
    n = 256 / 512 parity cases exercised."""
    if len(_covered) < 8:
        pytest.skip("needs test_hierarchy_matches_oracle_at_scale in the same session")
    covered = set().union(*_covered.values())
    cfg = wl.CONFIGS[4]
    n = cfg.n
    ctx = make_ctx(n)
    h, A = wl.ice_fields(cfg)
    va = wl.wind_nodal(n, cfg.dt, cfg.moving)
    vo = wl.ocean_nodal(n)
    v0 = torch.zeros(ctx.N, dtype=torch.float64, device="cuda")
    ctx.set_step(cfg.dt, cfg.dt, h, A, v0, va, vo)
    vv = v0.clone()
    for _ in range(6):
        ctx.newton_step(vv)
    hits = ctx.spgemm_path_hits()
    used = {PATHS[k] for k, c in enumerate(hits) if c}
    assert used <= covered, (used, covered)
    print("config 4 spgemm paths", sorted(used), "covered", sorted(covered))


@pytest.mark.parametrize("n", [64, 128])
def test_problem1_parity(n):
    """PAPER.md Problem I (analytic A/H with narrow bands, v_a = (5, 5) m/s, v_o = 0,
    f_c = 0, the paper's 1e4 residual reduction): the product path (AMG-FGMRES) and the
    oracle (direct solves) agree on the Newton count (+-1) and the converged velocity (1e-8).
    These are the hardest inputs in the repo (A down to ~0.1, zeta over > 10 decades)."""
    inp = wl.problem1_inputs(n)
    prm = wl.PhysParams(f_c=0.0)
    vo, _, ho = newton.solve_step(inp, prm, rtol=1e-4)
    assert ho["converged"]
    ctx = make_ctx(n, f_c=0.0, newton_rtol=1e-4, krylov_rtol=1e-10)
    vg, st = ctx.solve_step(inp.dt, inp.t_new, inp.h, inp.A, inp.v_prev, inp.v_air, inp.v_ocean)
    assert st["converged"] == 1, st
    assert abs(st["newton_iters"] - ho["newton_iters"]) <= 1, (st["newton_iters"], ho["newton_iters"])
    assert np.linalg.norm(np_(vg) - vo) <= 1e-8 * np.linalg.norm(vo)


@pytest.mark.parametrize("n,lag", [(32, 0), (64, 10), (64, 4)])
def test_newton_ew_lagged_hierarchy_matches_oracle(n, lag):
    """Product defaults (Eisenstat-Walker forcing, reading G29) with the lagged hierarchy of
    reading G31 (amg_lag): GPU and oracle tier B (same AMG definition, same forcing and
    rebuild rules) agree on the Newton count (+-1), the Krylov total (+-10 %), the number of full
    AMG setups (+-1) and the converged velocity (1e-8), over two moving-cyclone steps."""
    cfg = wl.Config(f"lag{n}", n, 2, 2, True)
    hA = wl.ice_fields(cfg)
    ctx = make_ctx(n, krylov_forcing=1, amg_lag=lag)
    vo_ = None
    vg = torch.zeros(ctx.N, dtype=torch.float64, device="cuda")
    for s in range(2):
        inp = wl.step_inputs(cfg, s, v_prev=vo_, h_A=hA)
        vo_, _, ho = newton.solve_step(inp, PRM, linsolve="amg_fgmres", forcing=1, amg_lag=lag)
        vin = vg.clone()
        vg, st = ctx.solve_step(inp.dt, inp.t_new, inp.h, inp.A, vin, inp.v_air, inp.v_ocean)
        assert st["converged"] == 1 and ho["converged"], (s, st)
        assert abs(st["newton_iters"] - ho["newton_iters"]) <= 1, (s, st["newton_iters"], ho["newton_iters"])
        ko = sum(k["iters"] for k in ho["krylov"])
        assert abs(st["krylov_iters_total"] - ko) <= 0.1 * ko + 2, (s, st["krylov_iters_total"], ko)
        so = sum(ho["amg_rebuilt"])
        assert abs(st["amg_setups"] - so) <= 1, (s, st["amg_setups"], so)
        if lag == 0:
            assert st["amg_setups"] == st["newton_iters"]
        assert np.linalg.norm(np_(vg) - vo_) <= 1e-8 * np.linalg.norm(vo_), s


@pytest.mark.parametrize("n", [64, 256])
def test_reused_hierarchy_matches_oracle(n):
    """Reading G32 (amg_reuse = 1): a setup after a full setup in the same time step keeps the
    aggregates and every pattern and recomputes the values (numeric-only SpGEMMs on the kept
    patterns and kernel choices).  Against oracle amg.setup(J2, v=v2, reuse=H1): same levels,
    identical aggregates, A_l and P_l to 1e-11 row-relative, and the same V-cycle."""
    inp, pb, v1, pi1 = _plastic_state(n, 31)
    v2 = 0.7 * v1 + wl.random_velocity(n, 33, amp=0.02)
    pi2 = pb.pi_consistent(v2)
    J1 = pb.jacobian(v1, pi1, "sv")
    J2 = pb.jacobian(v2, pi2, "sv")
    H1 = OA.setup(J1, pb, v=v1)
    H2 = OA.setup(J2, pb, v=v2, reuse=H1)
    assert H2["reused"]
    ctx = make_ctx(n, amg_reuse=1)
    ctx.set_inputs(inp)
    ctx.assemble_jacobian(v1, pi1.ravel(), want_csr=False)
    ctx.amg_setup()
    hits0 = sum(ctx.spgemm_path_hits())
    ctx.assemble_jacobian(v2, pi2.ravel(), want_csr=False)
    nlev, _ = ctx.amg_setup()
    assert sum(ctx.spgemm_path_hits()) == hits0  # no symbolic SpGEMM ran: the patterns were kept
    assert nlev == len(H2["levels"])
    for l in range(nlev):
        A, P, agg = ctx.amg_level(l)
        assert rows_close(bsr_to_scipy(A), H2["levels"][l]["A"], 1.0) <= 1e-11, l
        if l < nlev - 1:
            assert np.array_equal(agg, H1["levels"][l]["agg"]), l
            assert rows_close(bsr_to_scipy(P), H2["levels"][l]["P"], 1.0) <= 1e-11, l
    # the V-cycle built on the reused hierarchy is the oracle's
    r = wl.random_interior_vector(n, 8)
    zo = OA.vcycle(H2, r)
    zg = np_(ctx.precond_apply(r))
    assert np.linalg.norm(zg - zo) <= 1e-9 * np.linalg.norm(zo)


@pytest.mark.parametrize("n", [32, 64])
def test_newton_ew_reused_aggregates_matches_oracle(n):
    """Product path with amg_reuse = 1 (reading G32) and Eisenstat-Walker forcing over two
    moving-cyclone steps: Newton count (+-1), Krylov total (+-10 %), the number of setups that
    kept the aggregates (+-1) and the converged velocity (1e-8) match oracle tier B."""
    cfg = wl.Config(f"reuse{n}", n, 2, 2, True)
    hA = wl.ice_fields(cfg)
    ctx = make_ctx(n, krylov_forcing=1, amg_reuse=1)
    vo_ = None
    vg = torch.zeros(ctx.N, dtype=torch.float64, device="cuda")
    for s in range(2):
        inp = wl.step_inputs(cfg, s, v_prev=vo_, h_A=hA)
        vo_, _, ho = newton.solve_step(inp, PRM, linsolve="amg_fgmres", forcing=1, amg_reuse=1)
        vin = vg.clone()
        vg, st = ctx.solve_step(inp.dt, inp.t_new, inp.h, inp.A, vin, inp.v_air, inp.v_ocean)
        assert st["converged"] == 1 and ho["converged"], (s, st)
        assert abs(st["newton_iters"] - ho["newton_iters"]) <= 1, (s, st["newton_iters"], ho["newton_iters"])
        ko = sum(k["iters"] for k in ho["krylov"])
        assert abs(st["krylov_iters_total"] - ko) <= 0.1 * ko + 2, (s, st["krylov_iters_total"], ko)
        ro = sum(ho["amg_reused"])
        assert abs(st["amg_reuses"] - ro) <= 1 and st["amg_reuses"] >= st["newton_iters"] - 2, (s, st, ro)
        assert np.linalg.norm(np_(vg) - vo_) <= 1e-8 * np.linalg.norm(vo_), s
