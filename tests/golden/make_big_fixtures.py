"""TEST INFRASTRUCTURE ONLY -- generates the BASELINE-size MG-CG fixtures (tests/golden/big_*.json).

Run here (CPU container; /root/reference present for the cfg2 reference run):
    python tests/golden/make_big_fixtures.py cfg2 cfg2o cfg3g cfg3r cfg5

  cfg2   257^3 Poisson, 7 levels, V(2,2), lanczos estimator, rtol 1e-8, seed 1234: the REFERENCE's
         own translation units + SPEC glue (oracle/_ref/tmg_ref_bench, built by oracle/build_ref.sh)
  cfg2o  the same problem through the C restatement (oracle/liboracle.so): pins the oracle at size
         (its x must hash equal to the reference's)
  cfg3g  513^3 variable coefficient (32 spheres, k = 1e4), 8 levels, V(3,3), Galerkin coarse
         operators (2^-3 P^T A P), oracle
  cfg3r  the same with rediscretised coarse operators (the reference default), oracle
  cfg5   129^3 x 3 Q1 elasticity, 6 levels, V(2,2), rtol 1e-6, elasticity oracle (no reference
         implementation exists; parity unpinned by the reference)

Each fixture records iterations, reason, ||x||_2, the final ||z||/||z0||, the preconditioned residual
history, a strided sample of x (natural order = 1-rank rank-block order) and the SHA-256 of x's bytes.
"""
from __future__ import annotations

import hashlib
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
OUT = os.environ.get("TMGX_FIXTURE_OUT", os.path.dirname(os.path.abspath(__file__)))  # e.g. gpurun_out/ on a big host
SEED_F, SEED_K = 1234, 7

CASES = {
    "cfg2": dict(np3=(257, 257, 257), nlevels=7, m=2, kind=0, galerkin=False, rtol=1e-8, stride=7919),
    "cfg2o": dict(np3=(257, 257, 257), nlevels=7, m=2, kind=0, galerkin=False, rtol=1e-8, stride=7919),
    "cfg3g": dict(np3=(513, 513, 513), nlevels=8, m=3, kind=1, galerkin=True, rtol=1e-8, stride=100003),
    "cfg3r": dict(np3=(513, 513, 513), nlevels=8, m=3, kind=1, galerkin=False, rtol=1e-8, stride=100003),
    "cfg5": dict(np3=(129, 129, 129), nlevels=6, m=2, kind=2, galerkin=False, rtol=1e-6, stride=2003),
}


def record(name, c, x, its, reason, hist, source, t):
    x = np.ascontiguousarray(x, dtype=np.float64)
    rec = {
        "case": name, "source": source, "np": list(c["np3"]), "nlevels": c["nlevels"], "m": c["m"],
        "kind": c["kind"], "galerkin": c["galerkin"], "rtol": c["rtol"], "seed_f": SEED_F, "seed_k": SEED_K,
        "estimator": "lanczos", "iterations": int(its), "reason": reason, "xnorm": float(np.linalg.norm(x)),
        "final_ratio": float(hist[-1] / hist[0]), "history": [float(v) for v in hist],
        "sample_stride": c["stride"], "x_sample": [float(v) for v in x[:: c["stride"]]],
        "x_sha256": hashlib.sha256(x.tobytes()).hexdigest(), "n": int(x.size), "wall_s": round(t, 1),
    }
    with open(os.path.join(OUT, f"big_{name}.json"), "w") as f:
        json.dump(rec, f, indent=0)
    print(name, its, reason, rec["xnorm"], rec["final_ratio"], f"{t:.0f}s", flush=True)


def run(name):
    c = CASES[name]
    t0 = time.time()
    if name == "cfg2":
        exe = os.path.join(ROOT, "oracle", "_ref", "tmg_ref_bench")
        dump = "/tmp/tmgx_fixture_x.bin"
        out = subprocess.run([exe, str(c["np3"][0]), str(c["nlevels"]), str(c["m"]), "1", "0", str(SEED_F),
                              "lanczos", "0", "0", dump], capture_output=True, text=True, check=True).stdout
        rep = json.loads(out.strip().splitlines()[-1])
        x = np.fromfile(dump, dtype=np.float64)
        os.unlink(dump)
        record(name, c, x, rep["iterations"], rep["reason"], rep["history"],
               "reference translation units + SPEC glue (oracle/_ref/tmg_ref_bench)", time.time() - t0)
        return
    from oracle import oracle as O

    if c["kind"] == 2:
        mg = O.ElastMG(c["np3"], c["nlevels"], smooth_its=c["m"])
        b = O.el_rhs(c["np3"])
        src = "elasticity oracle (oracle/tmg_elast_oracle.c)"
    else:
        mg = O.MG(c["np3"], c["nlevels"], kind=c["kind"], smooth_its=c["m"], seed_k=SEED_K,
                  galerkin=c["galerkin"])
        b = O.rhs(c["np3"], SEED_F)
        src = "C restatement (oracle/tmg_oracle.c)"
    x, rep = mg.solve(b, rtol=c["rtol"])
    record(name, c, x, rep["iterations"], rep["reason"], rep["history"], src, time.time() - t0)


if __name__ == "__main__":
    for n in sys.argv[1:] or ["cfg2", "cfg2o", "cfg5"]:
        run(n)
