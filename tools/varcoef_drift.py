"""Measured drift of the performance build (FMA contraction, tree reductions) against the oracle
on the rediscretised 1e4-contrast variable-coefficient solves of tests/test_gpu_parity.py::
test_mgcg_varcoef: iteration counts, and at equal iteration counts the max-norm relative and
2-norm relative solution differences. Prints one JSON line per case."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1604_07163_b200 import tmgx as T  # noqa: E402

for np3, nl, m in [((33, 33, 33), 4, 3), ((65, 65, 33), 5, 2)]:
    om = O.MG(np3, nl, kind=O.VARCOEF7, smooth_its=m, est_mode=O.EST_LANCZOS, seed_k=7)
    b = O.rhs(np3, 1234)
    xo, orep = om.solve(b, rtol=1e-8)
    w = T.World(1)
    s = T.SolverNode(w, T.Problem(np3, T.VARCOEF7_HARMONIC, seed_k=7), T.MGConfig(nl, m, T.EST_LANCZOS))
    x, rep = s.solve(b, cfg=T.KrylovConfig("cg", rtol=1e-8))
    its_o = orep["iterations"]
    if rep.iterations != its_o:
        xo2, _ = om.solve(b, rtol=0.0, max_its=rep.iterations)
    else:
        xo2 = xo
    print(json.dumps({"np3": np3, "nlevels": nl, "m": m, "its_gpu": rep.iterations, "its_oracle": its_o,
                      "maxrel_equal_its": float(np.max(np.abs(x - xo2)) / np.max(np.abs(xo2))),
                      "l2rel_equal_its": float(np.linalg.norm(x - xo2) / np.linalg.norm(xo2)),
                      "l2rel_vs_converged_oracle": float(np.linalg.norm(x - xo) / np.linalg.norm(xo))}), flush=True)
