"""cfg3 with rediscretised coarse operators (the reference default) at the full 513^3 size: the
parity build (bitwise equal to the C oracle at every size the oracle can run here, e.g. the
~370-iteration 33^3 / 65x65x33 var-coef solves) gives the reference algorithm's iteration count
and solution; the performance build is compared with it (iterations +-1, 1e-9 at equal counts).
Writes one JSON line."""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import SEED_F, SEED_K  # noqa: E402
from paper_1604_07163_b200 import tmgx as T  # noqa: E402

np3, nl, m = (513, 513, 513), 8, 3
torch.cuda.set_device(0)
out = {"case": "cfg3r", "np": list(np3), "nlevels": nl, "m": m, "galerkin": False}
xs = {}
for parity in (True, False):
    w = T.World(1, parity=parity)
    s = T.SolverNode(w, T.Problem(np3, T.VARCOEF7_HARMONIC, seed_k=SEED_K), T.MGConfig(nl, m, T.EST_LANCZOS))
    b = s.rhs(SEED_F)
    t0 = time.time()
    x, rep = s.solve(b, cfg=T.KrylovConfig("cg", rtol=1e-8, max_its=5000, initial_guess_nonzero=False))
    tag = "parity" if parity else "perf"
    out[tag] = {"iterations": rep.iterations, "reason": rep.reason, "xnorm": float(np.linalg.norm(x)),
                "x_sha256": hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest(),
                "final_ratio": float(rep.residual_history[-1] / rep.residual_history[0]),
                "wall_s": round(time.time() - t0, 1), "history_tail": [float(v) for v in rep.residual_history[-6:]]}
    xs[tag] = x
    del s, w
out["perf_vs_parity_rel2"] = float(np.linalg.norm(xs["perf"] - xs["parity"]) / np.linalg.norm(xs["parity"]))
print(json.dumps(out), flush=True)
