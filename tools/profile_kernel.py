"""Launch one kernel of the hot path (tmgx_bench_kernel `which` on `level`) a few times for an
ncu capture: python tools/profile_kernel.py WHICH [LEVEL] [CONFIG]."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import CONFIGS, GALERKIN  # noqa: E402
from paper_1604_07163_b200 import tmgx as T  # noqa: E402

which = int(sys.argv[1])
cfgname = sys.argv[3] if len(sys.argv) > 3 else "cfg2"
np3, nl, m, kind, tele, rtol = CONFIGS[cfgname]
level = int(sys.argv[2]) if len(sys.argv) > 2 else nl - 1
torch.cuda.set_device(0)
w = T.World(1)
s = T.SolverNode(w, T.Problem(np3, kind), T.MGConfig(nl, m, T.EST_LANCZOS, galerkin=GALERKIN.get(cfgname, False)))
ms, by = s.bench_kernel(which, level, iters=3)
print(f"kernel {which} level {level}: {ms*1e3:.1f} us, {by/ms/1e6:.0f} GB/s")
