"""Generates tests/golden/ref_mgcg.json from the reference's own compiled translation units
(oracle/_ref/tmg_ref_bench, built by oracle/build_ref.sh from /root/reference). Run in the
build container (the reference is not on the GPU box); the JSON is committed.

Each case: the reference solve's CG iterations, ||x||_2, final ||z||/||z0|| and the sha256 of
the solution bytes (rank-block order == natural order on one rank)."""
import hashlib
import json
import os
import subprocess
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "..", "..", "oracle", "_ref", "tmg_ref_bench")

# (N, levels, m, seed, estimator, galerkin, kind)
CASES = [
    (33, 4, 2, 42, "lanczos", 0, 0), (65, 5, 2, 42, "lanczos", 0, 0), (65, 5, 3, 42, "lanczos", 0, 0),
    (33, 4, 2, 42, "reference", 0, 0), (65, 5, 2, 42, "reference", 0, 0),
    (33, 4, 2, 42, "lanczos", 1, 0), (65, 5, 2, 42, "lanczos", 1, 0), (65, 5, 2, 42, "reference", 1, 0),
    (33, 4, 3, 1234, "lanczos", 0, 1), (33, 4, 3, 1234, "lanczos", 1, 1), (33, 4, 2, 1234, "reference", 1, 1),
    (17, 3, 2, 7, "lanczos", 0, 1), (17, 3, 1, 7, "lanczos", 0, 0),
]


def run(case):
    N, nl, m, seed, est, gal, kind = case
    with tempfile.TemporaryDirectory() as td:
        dump = os.path.join(td, "x.bin")
        out = subprocess.run([BIN, str(N), str(nl), str(m), "1", "0", str(seed), est, str(gal), str(kind), dump],
                             capture_output=True, text=True, check=True).stdout
        rec = json.loads(out.strip().splitlines()[-1])
        rec["x_sha256"] = hashlib.sha256(open(dump, "rb").read()).hexdigest()
    rec.pop("t_setup_s")
    rec.pop("t_solve_s")
    rec.update(dict(N=N, nlevels=nl, m=m, seed=seed, est=est, galerkin=gal, kind=kind))
    return rec


if __name__ == "__main__":
    recs = [run(c) for c in CASES]
    with open(os.path.join(HERE, "ref_mgcg.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_ref_golden.py (oracle/_ref/tmg_ref_bench: reference TUs + "
                                "SPEC glue)", "cases": recs}, f, indent=1)
    print(len(recs), "cases")
