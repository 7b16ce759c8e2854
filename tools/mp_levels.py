"""Per-level V-cycle profile of a BASELINE layout run as P processes sharing one B200 (the
multi-process data plane of one process per GPU, emulated): exact per-level peer bytes (what the
halos and telescope transfers would put on NVLink with one process per GPU) and per-level device
time (NOT representative of 8 GPUs: the processes time-share one GPU and every exchange waits on a
host barrier). usage: python tools/mp_levels.py cfg4|cfg2|cfg3 P  -> one JSON line."""
import json
import multiprocessing as mp
import os
import secrets
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(job, P, proc, cfg, q):
    try:
        from bench import GALERKIN, resolve
        from paper_1604_07163_b200 import tmgx as T

        np3, nl, m, kind, stages, rtol, _ = resolve(cfg, P)
        w = T.World(n_ranks=P, nproc=P, proc=proc, device=0, job=job)
        s = T.SolverNode(w, T.Problem(np3, kind), T.MGConfig(nl, m, T.EST_LANCZOS, galerkin=GALERKIN.get(cfg, False),
                                                              telescope=[T.TelescopeStage(*t) for t in stages]))
        prof = s.level_profile(reps=3)
        q.put((proc, prof))
        del s
        w.close()
    except Exception as e:  # noqa: BLE001
        q.put((proc, repr(e)))


def main():
    cfg, P = sys.argv[1], int(sys.argv[2])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    job = "lv" + secrets.token_hex(8)
    ps = [ctx.Process(target=worker, args=(job, P, p, cfg, q)) for p in range(P)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=1800) for _ in ps)
    for p in ps:
        p.join(timeout=120)
    bad = {p: v for p, v in out.items() if isinstance(v, str)}
    if bad:
        print(json.dumps({"cfg": cfg, "P": P, "error": bad}))
        return
    levels = []
    for i, lv in enumerate(out[0]):
        levels.append({"node": i, "kind": lv["kind"], "npoints": lv["npoints"], "ranks": lv["ranks"],
                       "peer_bytes_all_procs": int(sum(out[p][i]["peer_bytes"] for p in range(P))),
                       "us_max_emulated": round(max(out[p][i]["us"] for p in range(P)), 1)})
    from bench import resolve

    np3, nl, m, kind, stages, rtol, _ = resolve(cfg, P)
    print(json.dumps({"cfg": cfg, "P": P, "grid": list(np3), "nlevels": nl, "telescope": stages, "levels": levels}))


if __name__ == "__main__":
    main()
