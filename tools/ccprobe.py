"""Coarse-level latency probe: per-level V-cycle profile and the device time of a full solve for
the current TMGX_* environment: python tools/ccprobe.py [CONFIG]."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import CONFIGS, GALERKIN, SEED_F  # noqa: E402
from paper_1604_07163_b200 import tmgx as T  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
np3, nl, m, kind, tele, rtol = CONFIGS[cfgname]
torch.cuda.set_device(0)
w = T.World(1)
s = T.SolverNode(w, T.Problem(np3, kind), T.MGConfig(nl, m, T.EST_LANCZOS, galerkin=GALERKIN.get(cfgname, False)))
cfg = T.KrylovConfig("cg", rtol=rtol)
for _ in range(3):
    rep = s.solve_seeded(SEED_F, cfg=cfg)
ts = []
for _ in range(5):
    rep = s.solve_seeded(SEED_F, cfg=cfg)
    ts.append(rep.t_solve_s * 1e3)
env = {k: v for k, v in os.environ.items() if k.startswith("TMGX_")}
print(json.dumps({"cfg": cfgname, "env": env, "its": rep.iterations, "ms_min": min(ts), "ms_med": sorted(ts)[2]}),
      flush=True)
prof = s.level_profile(reps=10)
print(json.dumps({"levels_us": [round(p["us"], 1) for p in prof]}), flush=True)
