"""Debug: V-cycle with the blocked smoother (TMGX_TB=1) vs the unfused path (TMGX_TB=0) in the
parity build; prints where they differ (i, j, k of the finest level)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1604_07163_b200 import tmgx as T  # noqa: E402

for np3, nl in (((33,) * 3, 4), ((65,) * 3, 5), ((17,) * 3, 3), ((9,) * 3, 2), ((65, 33, 129), 4), ((129,) * 3, 5), ((65, 65, 33), 4)):
    n = np3[0]
    b = O.rhs(np3, 42)
    res = {}
    for tb in ("0", "1"):
        os.environ["TMGX_TB"] = tb
        w = T.World(1, parity=True)
        s = T.SolverNode(w, T.Problem(np3, T.POISSON7), T.MGConfig(nl, 2, T.EST_LANCZOS))
        res[tb] = s.pc_apply(b)
    d = np.nonzero(res["0"] != res["1"])[0]
    print(np3, nl, "mismatches", d.size, "max rel", np.max(np.abs(res["0"] - res["1"])) / np.max(np.abs(res["0"])))
    if d.size:
        i, j, k = d % np3[0], (d // np3[0]) % np3[1], d // (np3[0] * np3[1])
        print("  i", np.unique(i)[:20], " j", np.unique(j)[:20], " k", np.unique(k)[:20])
