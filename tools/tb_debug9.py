import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from oracle import oracle as O
from paper_1604_07163_b200 import tmgx as T
os.environ["TMGX_TB"] = "1"
os.environ["TMGX_GRAPHS"] = "0"
np3 = (9, 9, 9)
w = T.World(1, parity=True)
s = T.SolverNode(w, T.Problem(np3, T.POISSON7), T.MGConfig(2, 2, T.EST_LANCZOS))
print(s.pc_apply(O.rhs(np3, 42))[:5])
