"""Worker processes for the multi-process tests (imported by spawned children)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def node_selftest(job, nproc, proc, rounds, q):
    from paper_1604_07163_b200 import tmgx as T

    try:
        q.put((proc, T.node_selftest(job, nproc, proc, rounds)))
    except Exception as e:  # noqa: BLE001
        q.put((proc, repr(e)))


def solve_slice(job, n_ranks, nproc, proc, case, q):
    """One process of a multi-process World on cuda:0: V-cycle and full MG-CG solve of the seeded
    problem; returns this process's slices (rank-block order) and the reports."""
    import numpy as np

    from paper_1604_07163_b200 import tmgx as T

    try:
        np3, nl, m, kind, tele, bounds, parity = case
        w = T.World(n_ranks=n_ranks, nproc=nproc, proc=proc, device=0, job=job, parity=parity)
        s = T.SolverNode(w, T.Problem(np3, kind),
                         T.MGConfig(nl, m, T.EST_LANCZOS, cheb_bounds=bounds,
                                    telescope=[T.TelescopeStage(*t) for t in tele]))
        b = s.rhs(1234)
        y = s.pc_apply(b)
        x, rep = s.solve(b, cfg=T.KrylovConfig("cg", rtol=1e-8, initial_guess_nonzero=False))
        us, by = s.exchange_timing(nl - 1, reps=20)
        bnds = [s.bounds(l) for l in range(1, nl)]
        q.put((proc, dict(y=y, x=x, its=rep.iterations, hist=np.asarray(rep.residual_history), us=us, bytes=by,
                          bounds=bnds)))
        del s
        w.close()
    except Exception as e:  # noqa: BLE001
        q.put((proc, repr(e)))


def elast_slice(job, n_ranks, nproc, proc, case, q):
    """One process of a multi-process World running the Q1 elasticity MG-CG: V-cycle and solve;
    returns the global-order vectors with this process's boxes filled (zeros elsewhere)."""
    import numpy as np

    from paper_1604_07163_b200 import tmgx as T

    try:
        n, nl, tele, parity = case
        w = T.World(n_ranks=n_ranks, nproc=nproc, proc=proc, device=0, job=job, parity=parity)
        s = T.ElastSolver(w, (n,) * 3, nl, smooth_its=2, telescope=[T.TelescopeStage(*t) for t in tele])
        b = s.rhs()
        y = s.pc_apply(b)
        x, rep = s.solve(b, cfg=T.KrylovConfig("cg", rtol=1e-6, initial_guess_nonzero=False))
        bnds = [s.bounds(l) for l in range(1, nl)]
        q.put((proc, dict(y=y, x=x, its=rep.iterations, hist=np.asarray(rep.residual_history), bounds=bnds)))
        del s
        w.close()
    except Exception as e:  # noqa: BLE001
        q.put((proc, repr(e)))
