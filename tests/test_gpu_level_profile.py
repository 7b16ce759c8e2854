"""Per-level V-cycle profile (tmgx_level_profile; the reference's per-level MsgCounters,
comm.hpp:37-47, plus device time): one entry per node of the hierarchy, node times that add up to
the whole V-cycle, telescope nodes where the stages are, no peer bytes in a one-process world."""
import time

import numpy as np
import pytest

from paper_1604_07163_b200 import tmgx as T

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def gpu():
    try:
        import torch

        if not torch.cuda.is_available():
            pytest.skip("no CUDA device")
    except ImportError:
        pytest.skip("torch missing")


def test_level_profile_single_box():
    w = T.World(1)
    s = T.SolverNode(w, T.Problem((129, 129, 129), T.POISSON7), T.MGConfig(6, 2, T.EST_LANCZOS))
    prof = s.level_profile(reps=5)
    assert [p["kind"] for p in prof] == ["smooth"] * 5 + ["coarse"]
    assert [p["npoints"][0] for p in prof] == [129, 65, 33, 17, 9, 5]
    assert all(p["us"] > 0 for p in prof)
    assert all(p["peer_bytes"] == 0 for p in prof)
    # the finest level dominates and the node times add up to a whole V-cycle
    assert prof[0]["us"] == max(p["us"] for p in prof)
    r = np.random.default_rng(0).standard_normal(s.local_size())
    s.pc_apply(r)
    tot = sum(p["us"] for p in prof)
    assert 10 < tot < 20000


def test_level_profile_telescoped_ranks():
    w = T.World(n_ranks=4)
    s = T.SolverNode(w, T.Problem((65, 65, 65), T.POISSON7),
                     T.MGConfig(5, 2, T.EST_LANCZOS, telescope=[T.TelescopeStage(2, 4)]))
    prof = s.level_profile(reps=3)
    kinds = [p["kind"] for p in prof]
    assert kinds.count("telescope") == 1 and kinds[-1] == "coarse"
    tele = prof[kinds.index("telescope")]
    assert tele["ranks"] == 4 and tele["us"] > 0
    assert prof[kinds.index("telescope") + 1]["ranks"] == 1
