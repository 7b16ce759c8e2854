"""Multi-process data plane on one GPU: P processes, each a World process owning R/P boxes, share
cuda:0 and exchange halos, telescope gathers/scatters and CG scalars through the production
transport (kernel stores into peers' CUDA-IPC mailboxes + stream-ordered host barriers; no kernel
waits on another process). The result must equal the single-process run with the same R boxes
bit for bit -- V-cycle and complete MG-CG solve -- because every kernel and every rank-ordered
reduction is independent of which process owns a box (reference transport being replaced:
comm.cpp:187-212 send/recv, ordered_fold_sum comm.cpp:338-351, ScatterPlan scatter_plan.cpp:40-114,
spmv halo dist_matrix.cpp:188-208).
"""
import json
import multiprocessing as mp
import os
import secrets

import numpy as np
import pytest

import _mp_worker as W
from paper_1604_07163_b200 import tmgx as T

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (name, np3, nlevels, m, kind, telescope stages (level, r[, override]), R, P)
CASES = [
    ("cfg2@4: r=4 at L2", (129, 129, 129), 6, 2, T.POISSON7, [(2, 4)], 4, 4),
    ("cfg3@8: var-coef V(3,3), r=8 at L3", (129, 129, 129), 6, 3, T.VARCOEF7_HARMONIC, [(3, 8)], 8, 8),
    ("cfg4 nested 8->2->1", (129, 129, 65), 6, 2, T.POISSON7, [(3, 4), (1, 2)], 8, 8),
    ("8 boxes on 2 processes", (65, 65, 65), 5, 2, T.POISSON7, [(1, 8)], 8, 2),
]


@pytest.fixture(scope="module", autouse=True)
def gpu():
    try:
        import torch

        if not torch.cuda.is_available():
            pytest.skip("no CUDA device")
    except ImportError:
        pytest.skip("torch missing")


def _multi(case, parity):
    _, np3, nl, m, kind, tele, R, P = case
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    job = "g" + secrets.token_hex(8)
    args = (np3, nl, m, kind, tele, None, parity)
    ps = [ctx.Process(target=W.solve_slice, args=(job, R, P, p, args, q)) for p in range(P)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=900) for _ in ps)
    for p in ps:
        p.join(timeout=120)
    for p in range(P):
        assert not isinstance(out[p], str), f"process {p}: {out[p]}"
    return out


@pytest.mark.parametrize("parity", [False, True])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_multiprocess_equals_single_process(case, parity):
    name, np3, nl, m, kind, tele, R, P = case
    out = _multi(case, parity)
    w = T.World(n_ranks=R, parity=parity)
    s = T.SolverNode(w, T.Problem(np3, kind),
                     T.MGConfig(nl, m, T.EST_LANCZOS, telescope=[T.TelescopeStage(*t) for t in tele]))
    b = s.rhs(1234)
    y1 = s.pc_apply(b)
    x1, r1 = s.solve(b, cfg=T.KrylovConfig("cg", rtol=1e-8, initial_guess_nonzero=False))
    for lv in range(1, nl):
        assert all(out[p]["bounds"][lv - 1] == s.bounds(lv) for p in range(P))
    y = np.concatenate([out[p]["y"] for p in range(P)])
    x = np.concatenate([out[p]["x"] for p in range(P)])
    assert np.array_equal(y, y1), "V-cycle differs from the single-process run"
    assert all(out[p]["its"] == r1.iterations for p in range(P))
    assert np.array_equal(out[0]["hist"], r1.residual_history)
    assert np.array_equal(x, x1), "solve differs from the single-process run"
    # record the per-exchange cost (pack + publishing barrier + unpack) of the finest halo
    rec = {"case": name, "parity": parity, "R": R, "P": P, "its": r1.iterations,
           "us_per_exchange": [out[p]["us"] for p in range(P)], "bytes_per_exchange": [out[p]["bytes"] for p in range(P)]}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "multiproc_exchange.jsonl"), "a") as f:
        f.write(json.dumps(rec) + "\n")


# Q1 elasticity (cfg5's layout, scaled): (name, n, nlevels, telescope stages, R, P)
ELAST_CASES = [
    ("elast cfg5@8: r=8 at L2", 65, 5, [(2, 8)], 8, 8),
    ("elast 8 boxes on 2 processes", 33, 4, [(1, 8)], 8, 2),
]


@pytest.mark.parametrize("parity", [False, True])
@pytest.mark.parametrize("case", ELAST_CASES, ids=[c[0] for c in ELAST_CASES])
def test_elast_multiprocess_equals_single_process(case, parity):
    """The elasticity V-cycle and solve over P processes equal the one-process run with the same
    R boxes bit for bit (halos and telescope transfers per component through the mailboxes,
    rank-ordered dot sums)."""
    name, n, nl, tele, R, P = case
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    job = "e" + secrets.token_hex(8)
    ps = [ctx.Process(target=W.elast_slice, args=(job, R, P, p, (n, nl, tele, parity), q)) for p in range(P)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=900) for _ in ps)
    for p in ps:
        p.join(timeout=120)
    for p in range(P):
        assert not isinstance(out[p], str), f"process {p}: {out[p]}"
    w = T.World(n_ranks=R, parity=parity)
    s = T.ElastSolver(w, (n,) * 3, nl, smooth_its=2, telescope=[T.TelescopeStage(*t) for t in tele])
    b = s.rhs()
    y1 = s.pc_apply(b)
    x1, r1 = s.solve(b, cfg=T.KrylovConfig("cg", rtol=1e-6, initial_guess_nonzero=False))
    for lv in range(1, nl):
        assert all(out[p]["bounds"][lv - 1] == s.bounds(lv) for p in range(P))
    y = sum(out[p]["y"] for p in range(P))
    x = sum(out[p]["x"] for p in range(P))
    assert np.array_equal(y, y1), "V-cycle differs from the single-process run"
    assert all(out[p]["its"] == r1.iterations for p in range(P))
    assert np.array_equal(out[0]["hist"], r1.residual_history)
    assert np.array_equal(x, x1), "solve differs from the single-process run"
