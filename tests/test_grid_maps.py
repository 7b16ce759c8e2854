"""CPU: product index maps (C++ behind the C-ABI) are bit-exact with the oracle restatement
of grid.cpp / comm.cpp (itself pinned by tests/test_oracle_pins.py)."""
import itertools

import numpy as np
import pytest

from oracle import oracle as O
from paper_1604_07163_b200 import tmgx as T

SHAPES = [(9, 9, 9), (17, 9, 5), (33, 33, 33), (65, 65, 33), (257, 257, 257), (513, 513, 257), (513, 257, 257),
          (129, 129, 129), (5, 5, 3)]


def same(h, oh):
    assert h.proc_grid == tuple(oh.pg)
    for a in range(3):
        assert list(h.axis_offsets[a]) == oh.offsets(a)


@pytest.mark.parametrize("np3", SHAPES)
@pytest.mark.parametrize("size", [1, 2, 3, 4, 6, 8, 12, 16])
def test_headers_coarsen(np3, size):
    try:
        oh = O.build_header(size, np3)
    except ValueError:
        with pytest.raises(T.ConfigError):
            T.create_grid_header(size, np3)
        return
    h = T.create_grid_header(size, np3)
    same(h, oh)
    assert list(h.layout()) == list(O.layout_offsets(oh))
    while True:
        oc = O.coarsen_header(oh)
        if oc is None:
            with pytest.raises(T.ConfigError):
                T.coarsen(h)
            break
        h, oh = T.coarsen(h), oc
        same(h, oh)


@pytest.mark.parametrize("size,r", [(8, 8), (8, 4), (8, 2), (6, 4), (4, 1), (4, 4), (2, 2), (8, 3), (12, 5)])
@pytest.mark.parametrize("np3", [(65, 65, 65), (65, 65, 33), (17, 17, 9), (33, 33, 33), (9, 9, 9)])
def test_telescope_maps(size, r, np3):
    try:
        oh = O.build_header(size, np3)
    except ValueError:
        return
    h = T.create_grid_header(size, np3)
    sp = T.split_strided(size, r)
    assert sp.member_map == O.split_strided(size, r)
    for ov in [(0, 0, 0), (1, 0, 0), (0, 0, 1)]:
        try:
            onh = O.repartition(oh, len(sp.member_map), ov)
        except ValueError:
            with pytest.raises(T.ConfigError):
                T.repartition_onto(h, sp, tuple(None if o == 0 else o for o in ov))
            continue
        nh = T.repartition_onto(h, sp, tuple(None if o == 0 else o for o in ov))
        same(nh, onh)
        assert list(T.prefusion_layout(nh, sp)) == list(O.prefusion_layout(onh, size, sp.member_map))
        if h.n_unknowns() <= 40000:
            assert np.array_equal(T.build_permutation(h, nh), O.build_permutation(oh, onh))


def test_natural_global_bijection():
    h = T.create_grid_header(6, (9, 17, 5))
    oh = O.build_header(6, (9, 17, 5))
    for g in range(h.n_unknowns()):
        n = h.global_to_natural(g)
        assert n == O.global_to_natural(oh, g)
        assert h.natural_to_global(n) == g
    perm = T.rank_block_to_natural(h)
    assert sorted(perm.tolist()) == list(range(h.n_unknowns()))
    assert all(perm[g] == O.global_to_natural(oh, g) for g in range(0, h.n_unknowns(), 13))
