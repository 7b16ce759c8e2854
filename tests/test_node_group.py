"""CPU, multi-process: the node-local process group behind the multi-process World
(tmgx_node.cpp: shared-memory barrier + allgather; the GPU path adds only CUDA IPC handles and
stream-ordered host barriers on top of it)."""
import multiprocessing as mp
import os
import secrets

import pytest

import _mp_worker as W
from paper_1604_07163_b200 import tmgx as T


def _run(nproc, rounds, procs=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    job = "t" + secrets.token_hex(8)
    ps = [ctx.Process(target=W.node_selftest, args=(job, nproc, p, rounds, q)) for p in (procs or range(nproc))]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    return out


@pytest.mark.parametrize("nproc", [2, 4, 8])
def test_barrier_allgather(nproc):
    out = _run(nproc, 100)
    for p in range(nproc):
        assert out[p] == (nproc * (nproc - 1) // 2, 100), out[p]


def test_missing_peer_times_out(monkeypatch):
    monkeypatch.setenv("TMGX_BARRIER_TIMEOUT", "2")
    out = _run(3, 5, procs=[0, 1])  # process 2 never joins
    for p in (0, 1):
        assert isinstance(out[p], str) and "barrier timed out" in out[p], out[p]


def test_bad_arguments():
    with pytest.raises(T.ConfigError):
        T.node_selftest("a/b", 2, 0, 1)
    with pytest.raises(T.ConfigError):
        T.node_selftest("ok", 2, 5, 1)
