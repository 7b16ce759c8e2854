"""GPU: the Q1 elasticity path split into boxes and telescoped (BASELINE configs[4]: 8 GPUs,
telescope reduction factor 8 at level 3).

The boxes are the scalar path's GridHeader boxes (choose_proc_grid, grid.cpp:209-240), the halos
its box halo (ghost_exchange, grid.cpp:645-696) per component, the telescope its gather /
scatter plans (TelescopePC). Every V-cycle operation is pointwise or a stencil
over halo-filled boxes, so with the Chebyshev intervals fixed the split and telescoped V-cycle
is bit for bit the one-box V-cycle of the elasticity oracle in the parity build. Solves differ
from the one-box solve only by the rank-ordered dot sums (ordered_fold_sum, comm.cpp:338-351):
iterations within 1, solution within 1e-9 (north_star bar).
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1604_07163_b200 import tmgx as T

pytestmark = pytest.mark.gpu
TOL_SOLUTION = 1e-9


@pytest.fixture(scope="module", autouse=True)
def gpu():
    try:
        import torch

        if not torch.cuda.is_available():
            pytest.skip("no CUDA device")
    except ImportError:
        pytest.skip("torch missing")


def rel(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


def oracle_bounds(om, nl):
    out = []
    for lv in range(nl):
        out += list(om.bounds(lv)) if lv > 0 else [0.1, 1.1]
    return out


# (ranks, levels, telescope stages): split down to the LU level (gathered there), one stage
# onto one box, nested 8 -> 2 -> 1, an uneven 6-box split
LAYOUTS = [
    (8, 17, 3, [T.TelescopeStage(0, 8)]),
    (8, 33, 4, [T.TelescopeStage(1, 8)]),
    (8, 33, 4, [T.TelescopeStage(2, 4), T.TelescopeStage(1, 2)]),
    (6, 33, 4, [T.TelescopeStage(2, 6)]),
]


@pytest.mark.parametrize("parity", [True, False])
@pytest.mark.parametrize("layout", range(len(LAYOUTS)))
def test_elast_boxes_vcycle_bitwise(parity, layout):
    R, n, nl, tele = LAYOUTS[layout]
    om = O.ElastMG((n,) * 3, nl, smooth_its=2)
    bounds = oracle_bounds(om, nl)
    w = T.World(R, parity=parity)
    s = T.ElastSolver(w, (n,) * 3, nl, smooth_its=2, telescope=tele, cheb_bounds=bounds)
    rng = np.random.default_rng(11 + layout)
    for level in range(nl):
        x = rng.standard_normal(om.level_size(level))
        y, yo = s.level_apply(level, x), om.apply(level, x)
        if parity:
            assert np.array_equal(y, yo), level
        else:
            assert rel(y, yo) < 1e-12, level
    b = rng.standard_normal(om.level_size(nl - 1))
    xs, xso = s.level_smooth(nl - 1, b), om.smooth(nl - 1, b)
    v, vo = s.pc_apply(b), om.vcycle(nl - 1, b)
    if parity:
        assert np.array_equal(xs, xso)
        assert np.array_equal(v, vo)
    else:
        assert rel(xs, xso) < 1e-11
        assert rel(v, vo) < 1e-10


@pytest.mark.parametrize("parity", [True, False])
def test_elast_boxes_telescoped_solve(parity):
    """33^3, 4 levels, 8 boxes telescoped r = 8 at level 1, estimated intervals: the CG solve
    matches the one-box oracle (iterations +-1, solution 1e-9)."""
    n, nl = 33, 4
    w = T.World(8, parity=parity)
    s = T.ElastSolver(w, (n,) * 3, nl, smooth_its=2, telescope=[T.TelescopeStage(1, 8)])
    om = O.ElastMG((n,) * 3, nl, smooth_its=2)
    for lv in range(1, nl):
        lo, hi = s.bounds(lv)
        olo, ohi = om.bounds(lv)
        assert abs(hi - ohi) / ohi < 1e-10 and abs(lo - olo) / olo < 1e-10
    b = O.el_rhs((n,) * 3)
    x, rep = s.solve(b, cfg=T.KrylovConfig("cg", rtol=1e-6))
    xo, orep = om.solve(b, rtol=1e-6)
    assert rep.converged()
    assert abs(rep.iterations - orep["iterations"]) <= 1
    if rep.iterations != orep["iterations"]:
        xo, orep = om.solve(b, rtol=0.0, max_its=rep.iterations)
    assert rel(x, xo) < TOL_SOLUTION


def test_elast_boxes_errors():
    w = T.World(8)
    with pytest.raises(T.ConfigError):  # LU on 8 ranks: no telescope stage reaches one rank
        T.ElastSolver(w, (17,) * 3, 3)
    with pytest.raises(T.ConfigError):
        T.ElastSolver(w, (17,) * 3, 3, telescope=[T.TelescopeStage(1, 8)], cheb_bounds=[0.1, 1.1])
