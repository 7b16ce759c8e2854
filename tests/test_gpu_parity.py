"""GPU parity: the sm_100a path (through the C-ABI) against the pinned CPU oracle.

Bar (BASELINE.json north_star): index maps bit-exact; CG iteration counts equal (or +-1);
solution relative difference <= 1e-9 in fp64. The parity build (-fmad=false) must reproduce
the oracle's stencil, smoother, transfer, coarse-solve and V-cycle arithmetic bit for bit;
the performance build (FMA contraction) within 1e-12 relative on those kernels.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1604_07163_b200 import tmgx as T

pytestmark = pytest.mark.gpu

TOL_KERNEL = 1e-12  # perf build vs oracle per kernel (FMA contraction only)
TOL_SOLUTION = 1e-9  # north_star: final solution relative agreement


def _need_gpu():
    try:
        import torch

        if not torch.cuda.is_available():
            pytest.skip("no CUDA device")
    except ImportError:
        pytest.skip("torch missing")


@pytest.fixture(scope="module", autouse=True)
def gpu():
    _need_gpu()


def rel(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


def check(a, b, parity):
    if parity:
        assert np.array_equal(a, b), f"not bitwise: max rel {rel(a, b):.3e}"
    else:
        assert rel(a, b) <= TOL_KERNEL, f"rel {rel(a, b):.3e}"


def make(np3, nlevels, kind=T.POISSON7, m=2, est=T.EST_LANCZOS, parity=False, n_ranks=1, bounds=None,
         telescope=(), hint=None, seed_k=7, galerkin=False):
    w = T.World(n_ranks=n_ranks, parity=parity)
    s = T.SolverNode(w, T.Problem(np3, kind, proc_grid_hint=hint, seed_k=seed_k),
                     T.MGConfig(nlevels, m, est, cheb_bounds=bounds, telescope=list(telescope), galerkin=galerkin))
    return w, s


def oracle_mg(np3, nlevels, kind=O.POISSON7, m=2, est=O.EST_LANCZOS, seed_k=7, galerkin=False):
    return O.MG(np3, nlevels, kind=kind, smooth_its=m, est_mode=est, seed_k=seed_k, galerkin=galerkin)


def oracle_bounds(mg, nlevels):
    b = np.zeros(2 * nlevels)
    for l in range(1, nlevels):
        b[2 * l], b[2 * l + 1] = mg.bounds(l)
    return b


KINDS = [(T.POISSON7, O.POISSON7), (T.VARCOEF7_HARMONIC, O.VARCOEF7)]


@pytest.mark.parametrize("parity", [True, False])
@pytest.mark.parametrize("kind", KINDS)
def test_operator_apply(parity, kind):
    np3, nl = (17, 33, 9), 3
    om = oracle_mg(np3, nl, kind[1])
    w, s = make(np3, nl, kind[0], parity=parity, bounds=oracle_bounds(om, nl))
    rng = np.random.default_rng(1)
    for level in range(nl):
        n = om.level_size(level)
        x = rng.standard_normal(n)
        check(s.level_apply(level, x), om.apply(level, x), parity)


@pytest.mark.parametrize("parity", [True, False])
@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("m", [1, 2, 3])
def test_smoother(parity, kind, m):
    np3, nl = (17, 17, 17), 3
    om = oracle_mg(np3, nl, kind[1], m=m)
    w, s = make(np3, nl, kind[0], m=m, parity=parity, bounds=oracle_bounds(om, nl))
    rng = np.random.default_rng(2)
    n = om.level_size(2)
    b = rng.standard_normal(n)
    check(s.level_smooth(2, b), om.smooth(2, b), parity)  # from x = 0
    x0 = rng.standard_normal(n)
    check(s.level_smooth(2, b, x0), om.smooth(2, b, x0), parity)


@pytest.mark.parametrize("parity", [True, False])
@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("zc", [None, "3", "64"])
def test_smoother_blocked_m3(parity, kind, zc, monkeypatch):
    """The temporally blocked V(3,3) smoother (k_cheb3_tb: three Chebyshev passes per kernel) on a
    level wide enough for it, odd extents, z-chunks of 1 plane (default split), 3 and all planes:
    bitwise the oracle in the parity build, 1e-12 in the performance build, from x = 0 and from
    a non-zero x."""
    if zc:
        monkeypatch.setenv("TMGX_TB_ZC", zc)
    np3, nl = (65, 41, 49), 3
    om = oracle_mg(np3, nl, kind[1], m=3)
    w, s = make(np3, nl, kind[0], m=3, parity=parity, bounds=oracle_bounds(om, nl))
    rng = np.random.default_rng(5)
    n = om.level_size(2)
    b = rng.standard_normal(n)
    check(s.level_smooth(2, b), om.smooth(2, b), parity)
    x0 = rng.standard_normal(n)
    check(s.level_smooth(2, b, x0), om.smooth(2, b, x0), parity)


@pytest.mark.parametrize("parity", [True, False])
def test_transfer_and_coarse(parity):
    np3, nl = (17, 33, 17), 3
    om = oracle_mg(np3, nl, O.VARCOEF7)
    w, s = make(np3, nl, T.VARCOEF7_HARMONIC, parity=parity, bounds=oracle_bounds(om, nl))
    rng = np.random.default_rng(3)
    n2, n1, n0 = om.level_size(2), om.level_size(1), om.level_size(0)
    b, x = rng.standard_normal(n2), rng.standard_normal(n2)
    r = b - om.apply(2, x)
    check(s.residual_restrict(2, b, x), om.restrict(2, r), parity)
    xc, xf = rng.standard_normal(n1), rng.standard_normal(n2)
    check(s.prolong_add(2, xc, xf), om.prolong_add(2, xc, xf), parity)
    bc = rng.standard_normal(n0)
    got, want = s.coarse_solve(bc), om.coarse_solve(bc)
    if parity:
        assert np.array_equal(got, want)
    else:  # explicit inverse from the same LU factors
        assert rel(got, want) < 1e-12


@pytest.mark.parametrize("parity", [True, False])
@pytest.mark.parametrize("kind", KINDS)
def test_vcycle(parity, kind):
    np3, nl = (33, 33, 33), 4
    om = oracle_mg(np3, nl, kind[1])
    w, s = make(np3, nl, kind[0], parity=parity, bounds=oracle_bounds(om, nl))
    b = O.rhs(np3, 42)
    got, want = s.pc_apply(b), om.vcycle(nl - 1, b)
    if parity:
        assert np.array_equal(got, want)
    else:
        assert rel(got, want) < 1e-11


@pytest.mark.parametrize("est", [T.EST_LANCZOS, T.EST_REFERENCE])
@pytest.mark.parametrize("kind", KINDS)
def test_estimator(est, kind):
    np3, nl = (33, 33, 33), 4
    om = oracle_mg(np3, nl, kind[1], est=est)
    w, s = make(np3, nl, kind[0], est=est)
    for l in range(1, nl):
        lo, hi = s.bounds(l)
        olo, ohi = om.bounds(l)
        assert abs(hi - ohi) / ohi < 1e-10 and abs(lo - olo) / olo < 1e-10


def test_rhs_bitwise():
    w, s = make((33, 17, 9), 2)
    assert np.array_equal(s.rhs(42), O.rhs((33, 17, 9), 42))


GOLDEN = [  # SURVEY.md §8(c) table, reproduced bitwise by the oracle
    ((33,) * 3, 4, 2, T.EST_LANCZOS, 10, 0.059938767310706596),
    ((65,) * 3, 5, 2, T.EST_LANCZOS, 10, 0.060110378198142883),
    ((65,) * 3, 5, 3, T.EST_LANCZOS, 6, 0.060110378065276547),
    ((33,) * 3, 4, 2, T.EST_REFERENCE, 52, 0.059938766918487769),
    ((65,) * 3, 5, 2, T.EST_REFERENCE, 60, 0.060110377849060662),
]


@pytest.mark.parametrize("parity", [False, True])
@pytest.mark.parametrize("np3,nl,m,est,its,xnorm", GOLDEN)
def test_mgcg_golden(parity, np3, nl, m, est, its, xnorm):
    w, s = make(np3, nl, m=m, est=est, parity=parity)
    b = O.rhs(np3, 42)
    x, rep = s.solve(b, cfg=T.KrylovConfig("cg", rtol=1e-8))
    assert rep.converged()
    assert abs(rep.iterations - its) <= 1
    # SURVEY §7 "parity vs reduction order": compare solutions at equal iteration counts
    # (oracle re-run with max_its = GPU iterations, rtol = 0 when the counts differ by one).
    om = oracle_mg(np3, nl, m=m, est=est)
    xo, orep = om.solve(b, rtol=1e-8 if rep.iterations == its else 0.0, max_its=rep.iterations)
    assert orep["iterations"] == rep.iterations
    if rep.iterations == its:
        assert abs(np.sqrt(np.dot(x, x)) - xnorm) / xnorm < TOL_SOLUTION
    if parity:  # serial-fold dots + unfused arithmetic: the whole solve is bitwise the oracle's
        assert rep.iterations == its
        assert np.array_equal(x, xo)
        assert np.array_equal(rep.residual_history, orep["history"])
        return
    # the reference (shipped) estimator gives a 5x too wide interval and ~50 iterations, which
    # amplifies reduction-order rounding; the solution bar stays 1e-9 for the fixed estimator
    tol = TOL_SOLUTION if est == T.EST_LANCZOS else 1e-8
    assert rel(x, xo) < tol
    if est == T.EST_LANCZOS:
        np.testing.assert_allclose(rep.residual_history, orep["history"], rtol=1e-6)
    else:  # late residuals of the badly smoothed run oscillate around 1e-10: compare vs ||z0||
        np.testing.assert_allclose(rep.residual_history, orep["history"], rtol=0, atol=1e-5 * orep["history"][0])


@pytest.mark.parametrize("parity", [True, False])
@pytest.mark.parametrize("np3,nl,m", [((33, 33, 33), 4, 3), ((65, 65, 33), 5, 2)])
def test_mgcg_varcoef(parity, np3, nl, m):
    """Variable coefficient (32 spheres, contrast 1e4) with rediscretised coarse operators:
    the reference algorithm needs hundreds of CG iterations here (SURVEY §7 'Var-coef with 1e4
    contrast'). The parity build reproduces the oracle solve bit for bit (iterations, history,
    solution); the FMA/tree-reduction build drifts by a few iterations over such long Krylov
    runs, so its bar is iterations within 2% and 1e-8 at equal iteration counts. Measured
    (tools/varcoef_drift.py, profiles/r04_varcoef_perf_drift.jsonl): 33^3 V(3,3) 362 vs 367
    iterations, 7.6e-10 max-rel at equal counts; 65x65x33 V(2,2) 1037 vs 1050, 7.2e-9 -- the
    north_star +-1 / 1e-9 bar holds for the Galerkin north-star problem (cfg3g, 49 its), not for
    these ~10^3-iteration rediscretised runs."""
    om = oracle_mg(np3, nl, O.VARCOEF7, m=m)
    b = O.rhs(np3, 1234)
    xo, orep = om.solve(b, rtol=1e-8)
    w, s = make(np3, nl, T.VARCOEF7_HARMONIC, m=m, parity=parity)
    x, rep = s.solve(b, cfg=T.KrylovConfig("cg", rtol=1e-8))
    assert rep.converged()
    if parity:
        assert rep.iterations == orep["iterations"]
        assert np.array_equal(x, xo)
        assert np.array_equal(rep.residual_history, orep["history"])
        return
    assert abs(rep.iterations - orep["iterations"]) <= max(1, orep["iterations"] // 50)
    if rep.iterations != orep["iterations"]:
        xo, orep = om.solve(b, rtol=0.0, max_its=rep.iterations)
    assert rel(x, xo) < 1e-8


def _decomposed(np3, nl, n_ranks, telescope=(), kind=T.POISSON7, m=2, hint=None):
    w, s = make(np3, nl, kind, m=m, n_ranks=n_ranks, telescope=telescope, hint=hint)
    h, _ = s.level_info(nl - 1)
    perm = T.rank_block_to_natural(h)
    return w, s, h, perm


@pytest.mark.parametrize("n_ranks,tele", [
    (2, ()), (4, ()), (8, ()),
    (8, (T.TelescopeStage(1, 8),)),
    (8, (T.TelescopeStage(2, 8),)),
    (4, (T.TelescopeStage(2, 4),)),
    (8, (T.TelescopeStage(2, 4), T.TelescopeStage(1, 2))),
    (8, (T.TelescopeStage(2, 2, (None, None, 1)), T.TelescopeStage(1, 4))),
    (6, (T.TelescopeStage(1, 6),)),
])
def test_decomposed_and_telescoped(n_ranks, tele):
    """Box decompositions over emulated ranks on one GPU (spawn_world-style), with single and
    nested telescoping: same iterations (+-1) and solution (1e-9) as the 1-rank oracle."""
    np3, nl = (33, 33, 33), 4
    if not tele:
        # an untelescoped multi-rank hierarchy cannot end in LU on more than one rank
        with pytest.raises(T.ConfigError):
            make(np3, nl, n_ranks=n_ranks)
        tele = (T.TelescopeStage(0, n_ranks),)
    w, s, h, perm = _decomposed(np3, nl, n_ranks, tele)
    b_nat = O.rhs(np3, 42)
    x, rep = s.solve(b_nat[perm], cfg=T.KrylovConfig("cg", rtol=1e-8))
    x_nat = np.empty_like(x)
    x_nat[perm] = x
    om = oracle_mg(np3, nl)
    xo, orep = om.solve(b_nat, rtol=1e-8)
    assert abs(rep.iterations - orep["iterations"]) <= 1
    if rep.iterations != orep["iterations"]:
        xo, orep = om.solve(b_nat, rtol=0.0, max_its=rep.iterations)
    assert rel(x_nat, xo) < TOL_SOLUTION


def test_vcycle_partition_independent_bitwise():
    """With fixed Chebyshev bounds the V-cycle has no reductions, and every kernel evaluates in
    natural order, so decomposed + telescoped V-cycles are bitwise equal to the 1-rank one."""
    np3, nl = (33, 33, 33), 4
    om = oracle_mg(np3, nl)
    bounds = oracle_bounds(om, nl)
    b_nat = O.rhs(np3, 42)
    w1, s1 = make(np3, nl, parity=True, bounds=bounds)
    y1 = s1.pc_apply(b_nat)
    assert np.array_equal(y1, om.vcycle(nl - 1, b_nat))
    w8, s8 = make(np3, nl, parity=True, n_ranks=8, bounds=bounds,
                  telescope=[T.TelescopeStage(2, 4), T.TelescopeStage(1, 2)])
    h, _ = s8.level_info(nl - 1)
    perm = T.rank_block_to_natural(h)
    y8 = s8.pc_apply(b_nat[perm])
    y8n = np.empty_like(y8)
    y8n[perm] = y8
    assert np.array_equal(y8n, y1)


def test_telescope_gather_scatter_maps():
    """Gather == P-hat^T x then ScatterPlan::to_sub (bitwise); scatter inverts it (AC3)."""
    np3, nl = (65, 65, 33), 3
    w, s = make(np3, nl, n_ranks=8, telescope=[T.TelescopeStage(1, 4), T.TelescopeStage(0, 2)])
    hp, n_par = s.level_info(2)  # outer level
    # stage 0 sits at level 1: parent header = outer level-1 header
    hp1 = T.coarsen(hp)
    sp = T.split_strided(8, 4)
    hn = T.repartition_onto(hp1, sp)
    assert hn.proc_grid == (1, 2, 1)
    n1 = hp1.n_unknowns()
    x_par = np.arange(n1, dtype=np.float64) * 0.5 + 1.0  # rank-block order of parent level 1
    y = s.telescope_gather(0, x_par, n1)
    cols = T.build_permutation(hp1, hn)
    want = np.empty(n1)
    want[cols] = x_par  # (P-hat^T x)[q] with q = cols[p]
    assert np.array_equal(y, want)
    back = s.telescope_scatter(0, y, n1)
    assert np.array_equal(back, x_par)


# ------------------------------------------------------------------------ Galerkin levels
@pytest.mark.parametrize("parity", [True, False])
@pytest.mark.parametrize("kind", KINDS)
def test_galerkin_operator_and_vcycle(parity, kind):
    """27-point Galerkin rows (2^-3 P^T A P) built on the device: operator, smoother and V-cycle
    bitwise equal to the oracle's ptap-semantics rows in the parity build."""
    np3, nl = (33, 17, 33), 4
    om = oracle_mg(np3, nl, kind[1], galerkin=True)
    w, s = make(np3, nl, kind[0], parity=parity, bounds=oracle_bounds(om, nl), galerkin=True)
    rng = np.random.default_rng(5)
    for level in range(nl):
        x = rng.standard_normal(om.level_size(level))
        check(s.level_apply(level, x), om.apply(level, x), parity)
    b = rng.standard_normal(om.level_size(2))
    check(s.level_smooth(2, b), om.smooth(2, b), parity)
    bf = O.rhs(np3, 42)
    got, want = s.pc_apply(bf), om.vcycle(nl - 1, bf)
    if parity:
        assert np.array_equal(got, want)
    else:
        assert rel(got, want) < 1e-11


@pytest.mark.parametrize("parity", [True, False])
@pytest.mark.parametrize("kind,np3,nl,m", [(KINDS[0], (65, 65, 65), 5, 2), (KINDS[1], (33, 33, 33), 4, 3),
                                           (KINDS[1], (65, 65, 33), 5, 2)])
def test_galerkin_solve(parity, kind, np3, nl, m):
    om = oracle_mg(np3, nl, kind[1], m=m, galerkin=True)
    b = O.rhs(np3, 1234)
    xo, orep = om.solve(b, rtol=1e-8)
    w, s = make(np3, nl, kind[0], m=m, parity=parity, galerkin=True)
    x, rep = s.solve(b, cfg=T.KrylovConfig("cg", rtol=1e-8))
    assert rep.converged()
    if parity:
        assert rep.iterations == orep["iterations"]
        assert np.array_equal(x, xo)
        return
    assert abs(rep.iterations - orep["iterations"]) <= 1
    if rep.iterations != orep["iterations"]:
        xo, orep = om.solve(b, rtol=0.0, max_its=rep.iterations)
    assert rel(x, xo) < TOL_SOLUTION


def test_galerkin_decomposed_telescoped_bitwise():
    """Galerkin rows computed box by box (halo-exchanged 27-plane operators) and moved by the
    telescope gather (C3(i): P-hat^T A P-hat + row fusion) give the 1-rank V-cycle bitwise."""
    np3, nl = (33, 33, 33), 4
    om = oracle_mg(np3, nl, O.VARCOEF7, galerkin=True)
    bounds = oracle_bounds(om, nl)
    b_nat = O.rhs(np3, 42)
    w1, s1 = make(np3, nl, T.VARCOEF7_HARMONIC, parity=True, bounds=bounds, galerkin=True)
    y1 = s1.pc_apply(b_nat)
    assert np.array_equal(y1, om.vcycle(nl - 1, b_nat))
    w8, s8 = make(np3, nl, T.VARCOEF7_HARMONIC, parity=True, n_ranks=8, bounds=bounds, galerkin=True,
                  telescope=[T.TelescopeStage(2, 4), T.TelescopeStage(1, 2)])
    h, _ = s8.level_info(nl - 1)
    perm = T.rank_block_to_natural(h)
    y8 = s8.pc_apply(b_nat[perm])
    y8n = np.empty_like(y8)
    y8n[perm] = y8
    assert np.array_equal(y8n, y1)


# ---------------------------------------------------------------- options-driven trees
@pytest.mark.parametrize("n_ranks,opts,direct", [
    # §3.3.1 truncation box (N = 4 levels here, nc = 4): telescope onto one rank + LU
    (4, "-pc_type mg -pc_mg_levels 4 -mg_coarse_pc_type telescope -mg_coarse_pc_telescope_reduction_factor 4 "
        "-mg_coarse_telescope_pc_type lu", dict(nlevels=4, telescope=[T.TelescopeStage(0, 4)])),
    # §3.3.2 repartitioned coarse grid (N1 = 2, N2 = 3, r = 8): 4 fused levels, Galerkin
    (8, "-pc_type mg -pc_mg_levels 2 -pc_mg_galerkin -mg_coarse_pc_type telescope "
        "-mg_coarse_pc_telescope_reduction_factor 8 -mg_coarse_telescope_pc_type mg "
        "-mg_coarse_telescope_pc_mg_levels 3 -mg_coarse_telescope_pc_mg_galerkin",
     dict(nlevels=4, telescope=[T.TelescopeStage(2, 8)], galerkin=True)),
])
def test_options_tree_solve_matches_direct(n_ranks, opts, direct):
    """build_solver_tree on the paper's boxes drives the same GPU hierarchy as the direct
    configuration: bitwise-identical solves in the parity build (SPEC.md:646 'instantiate without
    error and solve the 3D Poisson fixture to rtol 1e-8')."""
    np3 = (33, 33, 33)
    dbo = T.OptionsDatabase(("-ksp_type cg -ksp_rtol 1e-8 " + opts).split(), parity=True)
    w = T.World(n_ranks=n_ranks, parity=True)
    s_opt, ksp = T.build_solver_tree(dbo, w, T.Problem(np3))
    assert dbo.unused() == []
    s_dir = T.SolverNode(w, T.Problem(np3), T.MGConfig(smooth_its=2, est_mode=T.EST_LANCZOS, **direct))
    h, _ = s_opt.level_info(direct["nlevels"] - 1)
    perm = T.rank_block_to_natural(h)
    b = O.rhs(np3, 42)[perm]
    x1, r1 = s_opt.solve(b, cfg=ksp)
    x2, r2 = s_dir.solve(b, cfg=T.KrylovConfig("cg", rtol=1e-8))
    assert r1.converged() and r1.iterations == r2.iterations
    assert np.array_equal(x1, x2)


def test_zero_initial_guess_ignores_x():
    """ksp_initial_guess_nonzero false (PETSc's default): x is output only, never read."""
    np3 = (33, 33, 33)
    w, s = make(np3, 4, parity=True)
    b = O.rhs(np3, 42)
    x0, r0 = s.solve(b, cfg=T.KrylovConfig("cg", rtol=1e-8))
    junk = np.full_like(b, np.nan)
    x1, r1 = s.solve(b, x=junk, cfg=T.KrylovConfig("cg", rtol=1e-8, initial_guess_nonzero=False))
    assert r1.iterations == r0.iterations and np.array_equal(x0, x1)


# ---------------------------------------------------------------- Q1 elasticity (configs[4])
def _elast(parity, n=17, nl=3, m=2):
    w = T.World(1, parity=parity)
    return w, T.ElastSolver(w, (n,) * 3, nl, smooth_its=m), O.ElastMG((n,) * 3, nl, smooth_its=m)


@pytest.mark.parametrize("parity", [True, False])
def test_elast_kernels(parity):
    w, s, om = _elast(parity)
    rng = np.random.default_rng(5)
    for level in range(3):
        x = rng.standard_normal(om.level_size(level))
        check(s.level_apply(level, x), om.apply(level, x), parity)
    for level in (1, 2):
        lo, hi = s.bounds(level)
        olo, ohi = om.bounds(level)
        if parity:
            assert (lo, hi) == (olo, ohi)
        else:
            assert abs(hi - ohi) / ohi < 1e-10
    b = rng.standard_normal(om.level_size(2))
    assert np.array_equal(s.rhs(), O.el_rhs((17,) * 3))
    if parity:
        check(s.level_smooth(2, b), om.smooth(2, b), True)
        check(s.pc_apply(b), om.vcycle(2, b), True)
    else:
        assert rel(s.level_smooth(2, b), om.smooth(2, b)) < 1e-11
        assert rel(s.pc_apply(b), om.vcycle(2, b)) < 1e-10


@pytest.mark.parametrize("parity", [True, False])
def test_elast_solve(parity):
    w, s, om = _elast(parity, n=33, nl=4)
    b = O.el_rhs((33,) * 3)
    x, rep = s.solve(b, cfg=T.KrylovConfig("cg", rtol=1e-6))
    xo, orep = om.solve(b, rtol=1e-6)
    assert rep.converged()
    if parity:
        assert rep.iterations == orep["iterations"] and np.array_equal(x, xo)
    else:
        assert abs(rep.iterations - orep["iterations"]) <= 1
        if rep.iterations != orep["iterations"]:
            xo, orep = om.solve(b, rtol=0.0, max_its=rep.iterations)
        assert rel(x, xo) < TOL_SOLUTION


def test_telescope_timing_table_schema():
    """Table-1 timing: T_setup from the plan build, T_apply = gather +
    scatter of the telescoped level on the device; both positive, bytes = 2 x 8 x level size."""
    w, s = make((33, 33, 33), 3, n_ranks=8, telescope=[T.TelescopeStage(2, 8)])
    t_setup, t_apply, by = s.telescope_timing(0, reps=5)
    assert t_setup > 0 and t_apply > 0 and by == 2 * 8 * 33 ** 3


@pytest.mark.parametrize("parity", [True, False])
def test_fused_residual_restrict_optin(parity, monkeypatch):
    """The opt-in fused residual + restriction kernel (TMGX_FUSE_RR=1, measured slower and off
    by default) keeps the restriction's arithmetic: bitwise in the parity build."""
    monkeypatch.setenv("TMGX_FUSE_RR", "1")
    monkeypatch.setenv("TMGX_FUSE_RR2", "0")
    np3, nl = (33, 65, 33), 3
    om = oracle_mg(np3, nl, O.VARCOEF7)
    w, s = make(np3, nl, T.VARCOEF7_HARMONIC, parity=parity, bounds=oracle_bounds(om, nl))
    rng = np.random.default_rng(9)
    n = om.level_size(nl - 1)
    b, x = rng.standard_normal(n), rng.standard_normal(n)
    check(s.residual_restrict(nl - 1, b, x), om.restrict(nl - 1, b - om.apply(nl - 1, x)), parity)


@pytest.mark.parametrize("np3,nl,kind", [((33, 65, 33), 3, 1), ((65, 65, 65), 4, 0), ((17, 33, 129), 3, 0),
                                         ((129, 17, 9), 3, 1), ((9, 9, 9), 2, 0)])
def test_separable_residual_restrict(np3, nl, kind, monkeypatch):
    """Performance build on single-box levels (default for constant-coefficient rows, TMGX_FUSE_RR2=2
    for variable-coefficient rows too): the separable fused residual + restriction
    (lane shuffle in x, one shared plane in y, register accumulator in z) against the oracle's
    restrict(b - A x) -- a different summation order, so within 1e-12 relative; every tile edge
    (31 x 4 coarse tiles, z chunks) and grid boundary is exercised by these shapes."""
    monkeypatch.setenv("TMGX_FUSE_RR2", "2")
    okind = O.VARCOEF7 if kind == 1 else O.POISSON7
    om = oracle_mg(np3, nl, okind)
    w, s = make(np3, nl, T.VARCOEF7_HARMONIC if kind == 1 else T.POISSON7, bounds=oracle_bounds(om, nl))
    rng = np.random.default_rng(13)
    n = om.level_size(nl - 1)
    b, x = rng.standard_normal(n), rng.standard_normal(n)
    got = s.residual_restrict(nl - 1, b, x)
    want = om.restrict(nl - 1, b - om.apply(nl - 1, x))
    assert rel(got, want) < 1e-12


@pytest.mark.parametrize("cfg", ["cfg2", "cfg5"])
def test_full_size_linearity_exact(cfg):
    """BASELINE sizes, size-independent property: scaling the right-hand side by 2 scales every
    intermediate of MG-CG exactly (powers of two commute with rounding), so the solve of 2b takes
    the same iterations and returns exactly 2x (257^3 Poisson; 129^3 x 3 elasticity)."""
    import bench as B

    np3, nl, m, kind, _, rtol = B.CONFIGS[cfg]
    cfgk = T.KrylovConfig("cg", rtol=rtol, initial_guess_nonzero=False)
    w = T.World(1)
    if kind == 2:
        s = T.ElastSolver(w, np3, nl, smooth_its=m)
        b = s.rhs()
    else:
        s = T.SolverNode(w, T.Problem(np3, kind), T.MGConfig(nl, m, T.EST_LANCZOS))
        b = s.rhs(B.SEED_F)
    x1, r1 = s.solve(b, cfg=cfgk)
    x2, r2 = s.solve(2.0 * b, cfg=cfgk)
    assert r1.converged() and r1.iterations == r2.iterations
    assert np.array_equal(x2, 2.0 * x1)


def test_vcycle_partition_independent_large():
    """129^3 (cfg5's grid, 6 levels): the 8-box, doubly telescoped V-cycle equals the 1-box one bit
    for bit (parity build, shared Chebyshev bounds) — the decomposition-invariance property at a
    size the CPU oracle cannot reach quickly."""
    np3, nl = (129, 129, 129), 6
    w1, s1 = make(np3, nl, parity=True)
    bounds = np.zeros(2 * nl)
    for l in range(1, nl):
        bounds[2 * l], bounds[2 * l + 1] = s1.bounds(l)
    w1, s1 = make(np3, nl, parity=True, bounds=bounds)
    b_nat = O.rhs(np3, 42)
    y1 = s1.pc_apply(b_nat)
    w8, s8 = make(np3, nl, parity=True, n_ranks=8, bounds=bounds,
                  telescope=[T.TelescopeStage(3, 4), T.TelescopeStage(1, 2)])
    h, _ = s8.level_info(nl - 1)
    perm = T.rank_block_to_natural(h)
    y8 = s8.pc_apply(b_nat[perm])
    y8n = np.empty_like(y8)
    y8n[perm] = y8
    assert np.array_equal(y8n, y1)
