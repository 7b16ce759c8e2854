"""A/B of the smoother paths on one level: per-kernel device time (tmgx_bench_kernel) and the
full solve time with the temporally blocked smoother on/off (TMGX_TB)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import CONFIGS, SEED_F  # noqa: E402
from paper_1604_07163_b200 import tmgx as T  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
np3, nl, m, kind, tele, rtol = CONFIGS[cfgname]
torch.cuda.set_device(0)
w = T.World(1)
s = T.SolverNode(w, T.Problem(np3, kind), T.MGConfig(nl, m, T.EST_LANCZOS))
cfg = T.KrylovConfig("cg", rtol=rtol)
out = {"tb": os.environ.get("TMGX_TB", "1"), "zc": os.environ.get("TMGX_TB_ZC", "32")}
for lvl in range(nl - 1, 0, -1):
    for which in (1, 3, 4, 5, 6, 7, 8, 9, 10, 11):
        try:
            ms, by = s.bench_kernel(which, lvl, iters=20)
            out[f"L{lvl}_k{which}"] = [round(ms * 1e3, 2), round(by / ms / 1e6, 1)]  # us, GB/s
        except Exception as e:  # noqa: BLE001
            out[f"L{lvl}_k{which}"] = str(e)[:60]
    if lvl < nl - 3:
        break
for _ in range(3):
    s.solve_seeded(SEED_F, cfg=cfg)
ts = []
for _ in range(10):
    rep = s.solve_seeded(SEED_F, cfg=cfg)
    ts.append(rep.t_solve_s * 1e3)
out["solve_ms"] = sorted(ts)[len(ts) // 2]
out["its"] = rep.iterations
print(json.dumps(out))
