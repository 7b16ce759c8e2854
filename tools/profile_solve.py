"""One steady-state MG-CG solve bracketed by cudaProfilerStart/Stop, for
`ncu --profile-from-start off` launch lists and full captures (profiles/)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import CONFIGS, GALERKIN, SEED_F, SEED_K  # noqa: E402
from paper_1604_07163_b200 import tmgx as T  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--max-its", type=int, default=10000)
args = ap.parse_args()
np3, nl, m, kind, tele, rtol = CONFIGS[args.config]
torch.cuda.set_device(0)
w = T.World(1)
s = T.SolverNode(w, T.Problem(np3, kind, seed_k=SEED_K),
                 T.MGConfig(nl, m, T.EST_LANCZOS, galerkin=GALERKIN.get(args.config, False)))
cfg = T.KrylovConfig("cg", rtol=rtol, max_its=args.max_its)
for _ in range(args.warmup):
    s.solve_seeded(SEED_F, cfg=cfg)
torch.cuda.synchronize()
torch.cuda.profiler.start()
rep = s.solve_seeded(SEED_F, cfg=cfg)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"its={rep.iterations} t={rep.t_solve_s*1e3:.3f} ms launches={rep.kernel_launches}")
