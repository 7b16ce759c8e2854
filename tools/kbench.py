"""Live kernel timings (CUDA events, tmgx_bench_kernel) on the finest level of a bench config:
python tools/kbench.py CONFIG ID [ID ...]  -> one JSON line per kernel."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import CONFIGS, GALERKIN  # noqa: E402
from paper_1604_07163_b200 import tmgx as T  # noqa: E402

cfgname = sys.argv[1]
np3, nl, m, kind, tele, rtol = CONFIGS[cfgname]
torch.cuda.set_device(0)
w = T.World(1)
s = T.SolverNode(w, T.Problem(np3, kind), T.MGConfig(nl, m, T.EST_LANCZOS, galerkin=GALERKIN.get(cfgname, False)))
tag = os.environ.get("KB_TAG", "")
for a in sys.argv[2:]:
    which, level = (int(a.split("@")[0]), int(a.split("@")[1])) if "@" in a else (int(a), nl - 1)
    ms, by = s.bench_kernel(which, level, iters=10)
    print(json.dumps({"cfg": cfgname, "tag": tag, "id": which, "level": level, "us": round(ms * 1e3, 1),
                      "GBs": round(by / ms / 1e6, 1)}), flush=True)
