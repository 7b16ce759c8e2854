"""Telescope setup/apply timing in the paper's Table 1 schema (SPEC.md
harness emit_csv columns n_C, N, r, T_setup_s, T_apply_s, T_solve_s, iterations, levels, ranks).

B200 single-GPU emulation: n_C reference ranks are boxes of one GPU's memory (the spawn_world
analogue), so the telescope's moves are on-device region copies, not NVLink transfers; the
finest level (N^3 vertices, 7-point Poisson, N = 2M+1) is telescoped by r and the rest of the
hierarchy runs on the sub-communicator. T_solve is one MG-CG solve to rtol 1e-8 (second of two).
usage: python tools/telescope_table.py [out.csv]
"""
import csv
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1604_07163_b200 import tmgx as T  # noqa: E402


def sig3(x):
    return f"{x:.2E}"


def run(n_c, n, r, nlevels):
    w = T.World(n_ranks=n_c)
    mg = T.MGConfig(nlevels=nlevels, smooth_its=2, est_mode=T.EST_LANCZOS,
                    telescope=[T.TelescopeStage(nlevels - 1, r)] + ([T.TelescopeStage(0, n_c // r)] if n_c // r > 1 else []))
    s = T.SolverNode(w, T.Problem((n, n, n)), mg)
    t_setup, t_apply, by = s.telescope_timing(0, reps=20)
    cfg = T.KrylovConfig("cg", rtol=1e-8)
    s.solve_seeded(1234, cfg=cfg)
    rep = s.solve_seeded(1234, cfg=cfg)
    return {"n_C": n_c, "N": n, "r": r, "T_setup_s": sig3(t_setup), "T_apply_s": sig3(t_apply),
            "T_solve_s": sig3(rep.t_solve_s), "iterations": rep.iterations, "levels": nlevels,
            "ranks": f"{n_c}->{n_c // r}" + ("->1" if n_c // r > 1 else ""), "apply_GBps": round(by / t_apply / 1e9, 1)}


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "telescope_table.csv")
    rows = []
    for n_c, grids in ((8, ((17, 3), (65, 5), (129, 6))), (64, ((17, 3), (65, 5), (129, 6)))):
        for n, nl in grids:
            for r in (2, 4, 8, 16, 32, 64):
                if r > n_c:
                    continue
                try:
                    rows.append(run(n_c, n, r, nl))
                except T.ConfigError as e:  # grid not decomposable on that sub-communicator
                    print(f"skip n_C={n_c} N={n} r={r}: {e}", flush=True)
                    continue
                print(rows[-1], flush=True)
    with open(out, "w", newline="") as f:
        wr = csv.DictWriter(f, fieldnames=list(rows[0].keys()))
        wr.writeheader()
        wr.writerows(rows)


if __name__ == "__main__":
    main()
