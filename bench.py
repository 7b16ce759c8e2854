"""MG-CG benchmark (BASELINE.json metric: MG-CG time-to-solution and DOF/s; smoother HBM GB/s).

Default workload (N=1): BASELINE configs[1] -- 3D constant-coefficient 7-point Poisson on
257^3 vertices, fp64, f = 2u-1 from seed, CG + 7-level MG V(2,2) Chebyshev(Jacobi), LU on 5^3,
rtol 1e-8. With N>1 processes (torchrun, one GPU each) the same global problem is box-split
over N GPUs and levels <= 3 are telescoped onto GPU 0 (reduction factor N): strong scaling.

One step = one complete MG-CG solve (setup, i.e. hierarchy + Chebyshev estimates, is outside
the timed region; this is the "second of two identical solves" protocol).
`value` = DOF/s with the right-hand side generated in HBM; `e2e` = DOF/s through the C-ABI
with pinned host b/x (H2D of b and x0, D2H of x inside the timed region).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (npoints, nlevels, smooth_its, kind, telescope_level, rtol)
    "cfg1": ((65, 65, 65), 5, 2, 0, None, 1e-8),
    "cfg2": ((257, 257, 257), 7, 2, 0, 3, 1e-8),
    "cfg3": ((513, 513, 513), 8, 3, 1, 4, 1e-8),
    "cfg4w": ((257, 257, 257), 7, 2, 0, 4, 1e-8),
    # Q1 elasticity, 3 dof/vertex (kind 2): N boxes, telescoped r = N at level 3 (BASELINE configs[4])
    "cfg5": ((129, 129, 129), 6, 2, 2, 3, 1e-6),
    # weak scaling, 257^3 per GPU (true-weak series): the global grid and the
    # nested telescope stages depend on N (resolve())
    "cfg4": ((257, 257, 257), 7, 2, 0, "nested", 1e-8),
}
CFG4_GRID = {1: (257, 257, 257), 2: (513, 257, 257), 4: (513, 513, 257), 8: (513, 513, 513)}


def resolve(config, world):
    """(np3, nlevels, m, kind, telescope stages [(level, r)], rtol, scaling) of a config at N."""
    np3, nlevels, m, kind, tele_level, rtol = CONFIGS[config]
    if config != "cfg4":
        stages = [(tele_level, world)] if (world > 1 and tele_level is not None) else []
        return np3, nlevels, m, kind, stages, rtol, "strong"
    if world not in CFG4_GRID:
        raise SystemExit(f"cfg4 is defined for 1, 2, 4, 8 GPUs (got {world})")
    np3 = CFG4_GRID[world]
    nlevels = 7 if world == 1 else 8
    # nested telescoping (BASELINE configs[3]): N -> 2 at level 4, 2 -> 1 at level 2
    stages = ([(4, world // 2)] if world > 2 else []) + ([(2, 2)] if world > 1 else [])
    return np3, nlevels, m, kind, stages, rtol, "weak"
# Coarse operators: rediscretised (reference default) for constant k;
# Galerkin 2^-3 P^T A P for the 1e4-contrast problem (with rediscretisation the reference
# algorithm needs ~500 CG iterations at 513^3).
GALERKIN = {"cfg3": True}
SEED_F = 1234
# CPU legs (cpu_baseline, --impl reference): problems above CPU_SAMPLE_MAX_DOF are timed on a
# bounded sample of at most CPU_SAMPLE_DOF vertices (cpu_reference_sample)
CPU_SAMPLE_MAX_DOF = 40_000_000
CPU_SAMPLE_DOF = 3_000_000
SEED_K = 7


def read_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device):
        self.device = device
        self.samples = []
        self._p = None
        self._lines = []
        self._t = None

    def _drain(self):
        for ln in self._p.stdout:
            self._lines.append(ln)

    def __enter__(self):
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                        "--format=csv,noheader,nounits", "-lms", "50"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._drain, daemon=True)
            self._t.start()
            time.sleep(0.3)  # first sample before the timed region
        except Exception:
            self._p = None
        return self

    def __exit__(self, *a):
        if self._p:
            time.sleep(0.1)
            self._p.terminate()
            try:
                self._p.wait(timeout=5)
            except Exception:
                self._p.kill()
            self._t.join(timeout=5)
        for ln in self._lines:
            v = [t.strip() for t in ln.split(",")]
            if len(v) == 7:
                self.samples.append(v)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}

        def num(s):
            try:
                return float(s)
            except ValueError:
                return None

        sm = [num(s[0]) for s in self.samples if num(s[0]) is not None]
        mx = [num(s[1]) for s in self.samples if num(s[1]) is not None]
        pw = [num(s[2]) for s in self.samples if num(s[2]) is not None]
        reasons = sorted({self.NAMES[i] for s in self.samples for i in range(4) if s[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples), "power_w_max": max(pw) if pw else None}


def workload_config(config, world, tele_level, galerkin, est):
    """The `config` object of both arms' JSON lines (identical for the same --config / N)."""
    np3, nlevels, m, kind, stages, rtol, _ = resolve(config, world)
    n_dof = np3[0] * np3[1] * np3[2]
    tele = bool(stages)
    return {"workload": f"{config}: {np3[0]}x{np3[1]}x{np3[2]} {'var-coef' if kind else 'Poisson'} {nlevels}-level "
                        f"MG V({m},{m}) Cheb-Jacobi CG rtol {rtol:g}, est={est}, "
                        f"coarse={'galerkin' if galerkin else 'rediscretised'}",
            "global_batch": 1, "seq_len": np3[0],
            "parallelism": f"box{world}" + "".join(f"+telescope(L{lv},r{r})" for lv, r in stages),
            "l2": ("inputs larger than L2 (one fine vector = %.0f MB)" % (n_dof * 8 / 1e6) if n_dof * 8 > 126e6 else
                   "L2-resident problem (one fine vector = %.1f MB): a latency benchmark" % (n_dof * 8 / 1e6))}


def cpu_reference_sample(config="cfg2", steps=1, warmup=0, galerkin=False, budget_s=0.0, world=1):
    """The reference algorithm on the host, on the SAME problem as the GPU arm (BASELINE config,
    full size): oracle/_ref (the reference's own translation units + the SPEC-following V-cycle
    glue) when it was built, else the C restatement in oracle/. One rank = one core (the
    reference has no threaded kernels; its n-rank mode is a mutex-serialised simulated transport).
    Setup (assembly, hierarchy, estimates) is excluded; `warmup` untimed solves first, then the
    mean over `steps` complete solves. Returns (dof_per_s, seconds_per_solve, kind, description,
    iterations)."""
    np3, nlevels, m, kind_p, _, rtol, _ = resolve(config, world)
    sample_note = "same problem as the GPU arm"
    if np3[0] * np3[1] * np3[2] > CPU_SAMPLE_MAX_DOF and os.environ.get("TMGX_REF_FULL", "0") != "1":
        # bounded sample (contract: the CPU leg must end within minutes): one complete solve of the
        # 513^3 / 8-level problem takes ~45 min on one core, so the same algorithm (operator kind,
        # V(m,m), coarse operators, rtol) runs at 129^3 with two levels fewer (the same 5^3 coarse
        # grid). DOF/s of the reference is size-independent to ~10% between 129^3 and 257^3 (cfg2).
        full = np3
        while np3[0] * np3[1] * np3[2] > CPU_SAMPLE_DOF and nlevels > 2:
            np3, nlevels = tuple((v - 1) // 2 + 1 for v in np3), nlevels - 1
        sample_note = (f"BOUNDED SAMPLE of the GPU arm's {full[0]}x{full[1]}x{full[2]} problem (TMGX_REF_FULL=1 "
                       f"times the full size): same operator and solver at")
    ref_bin = os.path.join(ROOT, "oracle", "_ref", "tmg_ref_bench")
    n = np3[0] * np3[1] * np3[2]
    if os.path.exists(ref_bin) and np3[0] == np3[1] == np3[2]:
        out = subprocess.run([ref_bin, str(np3[0]), str(nlevels), str(m), str(steps), str(warmup), str(SEED_F),
                              "lanczos", "1" if galerkin else "0", str(kind_p), "-", str(budget_s)],
                             capture_output=True, text=True, check=True).stdout
        rec = json.loads(out.strip().splitlines()[-1])
        t, its, kind = rec["t_solve_s"], rec["iterations"], "reference"
        setup, steps = rec["t_setup_s"], rec.get("steps_timed", steps)
    else:
        os.environ.setdefault("OMP_NUM_THREADS", "1")  # the port's element loops are OpenMP
        from oracle import oracle as O

        t0 = time.perf_counter()
        mg = O.MG(np3, nlevels, kind=kind_p, smooth_its=m, est_mode=O.EST_LANCZOS, seed_k=SEED_K,
                  galerkin=galerkin)
        b = O.rhs(np3, SEED_F)
        setup = time.perf_counter() - t0
        tw = 0.0
        for _ in range(warmup):
            t0 = time.perf_counter()
            mg.solve(b, rtol=rtol)
            tw = time.perf_counter() - t0
        if budget_s > 0 and tw > 0:
            steps = max(1, min(steps, int(budget_s // tw)))
        ts = []
        for _ in range(steps):
            t0 = time.perf_counter()
            _, rep = mg.solve(b, rtol=rtol)
            ts.append(time.perf_counter() - t0)
        t, its, kind = sum(ts) / len(ts), rep["iterations"], "port"
    impl = ("reference translation units + SPEC glue (oracle/_ref/tmg_ref_bench)" if kind == "reference"
            else "oracle C restatement (oracle/liboracle.so)")
    desc = (f"{sample_note}: {np3[0]}x{np3[1]}x{np3[2]}, {nlevels}-level MG V({m},{m}) CG rtol "
            f"{rtol:g}, {its} its; {steps} timed complete solve(s) after {warmup} untimed, setup ({setup:.1f} s) "
            f"excluded; 1 rank on 1 core; {impl}")
    return n / t, t, kind, desc, its, steps


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU implementation of the path on this host, on the
    GPU arm's config (same problem, same size). One complete 257^3 solve takes ~50 s on one
    core, so K steps are capped by a time budget (TMGX_REF_BUDGET_S, default 150 s of timed
    solves after one untimed solve); `steps` reports the solves actually timed."""
    np3, nlevels, m, kind, stages, rtol, scaling = resolve(args.config, world)
    tele_level = stages[0][0] if stages else None
    if rank != 0:
        return
    galerkin = GALERKIN.get(args.config, False) if args.galerkin is None else args.galerkin == "on"
    budget = float(os.environ.get("TMGX_REF_BUDGET_S", "150"))
    W = 1 if args.warmup > 0 else 0  # the reference protocol: time the second of identical solves
    rate, t, kind_s, desc, its, K = cpu_reference_sample(args.config, steps=max(args.steps, 1), warmup=W,
                                                         galerkin=galerkin, budget_s=budget if W else 0.0,
                                                         world=world)
    line = {
        "impl": "reference", "metric": "MG-CG DOF/s (time-to-solution)", "value": rate, "unit": "DOF/s",
        "n_gpus": args.gpus, "steps": K, "warmup": W, "steps_requested": args.steps,
        "warmup_requested": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded RHS, natural-index hash; BASELINE configs are synthetic)",
        "config": workload_config(args.config, world, tele_level, galerkin, args.est),
        "solve": {"iterations": its},
        "cpu_baseline": {"value": rate, "unit": "DOF/s", "cores": 1, "kind": kind_s, "sample": desc},
        "e2e": {"value": rate, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_elast(args, world, rank, local, np3, nlevels, m, rtol, stages, dist):
    """BASELINE configs[4]: Q1 elasticity MG-CG (ElastSolver). One box per GPU; with N > 1 the
    levels <= 3 are telescoped onto GPU 0 (reduction factor N). value = DOF/s with b, x resident in
    HBM; e2e through tmgx_elast_solve with pinned host b / x. Device times: max over ranks."""
    import torch

    from paper_1604_07163_b200 import tmgx as T

    job = None
    if world > 1:  # node-local rendezvous name for the peer-memory transport
        obj = [T.job_token() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        job = obj[0]

    def max_over_ranks(v):
        if not dist:
            return v
        t = torch.tensor([v], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    w = T.World(n_ranks=world, nproc=world, proc=rank, device=local, job=job)
    t0 = time.perf_counter()
    s = T.ElastSolver(w, np3, nlevels, smooth_its=m, telescope=[T.TelescopeStage(lv, r) for lv, r in stages])
    t_setup = time.perf_counter() - t0
    b_np = s.rhs()
    n_dof = b_np.size
    cfg = T.KrylovConfig("cg", rtol=rtol, initial_guess_nonzero=False)
    b_dev = torch.from_numpy(b_np).cuda()
    x_dev = torch.zeros_like(b_dev)
    for _ in range(max(args.warmup, 0)):
        rep = s.solve_ptr(b_dev.data_ptr(), x_dev.data_ptr(), cfg)
    barrier()
    dev_t, its = 0.0, 0
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            rep = s.solve_ptr(b_dev.data_ptr(), x_dev.data_ptr(), cfg)
            dev_t += rep.t_solve_s
            its = rep.iterations
        barrier()
    dev_t = max_over_ranks(dev_t)
    b_host = torch.from_numpy(b_np).pin_memory()
    x_host = torch.zeros(n_dof, dtype=torch.float64).pin_memory()
    s.solve_ptr(b_host.data_ptr(), x_host.data_ptr(), cfg)
    barrier()
    e2e_t = 0.0
    for _ in range(args.steps):
        t1 = time.perf_counter()
        s.solve_ptr(b_host.data_ptr(), x_host.data_ptr(), cfg)
        e2e_t += time.perf_counter() - t1
    barrier()
    e2e_t = max_over_ranks(e2e_t)
    ms, by, fl = s.bench_apply(20)
    ms = max_over_ranks(ms)
    if rank != 0:
        return
    # k_el_apply is fp64-FMA bound (576 FMAs per vertex): the roofline is the B200 fp64 vector
    # peak. MEASURED_PEAKS.json has none; profiles/r04_fp64_peak.json holds the one measured on
    # this pool's B200 (tools/fp64_peak: 8 independent DFMA chains per thread, full occupancy),
    # else the nominal 148 SMs x 64 DFMA/clk x 2 flop x 1.965 GHz = 37.2 TFLOP/s.
    fp64_peak, fp64_kind = 148 * 64 * 2 * 1.965e9 / 1e12, "nominal (148 SMs x 64 DFMA/clk x 1.965 GHz)"
    try:
        with open(os.path.join(ROOT, "profiles", "r04_fp64_peak.json")) as f:
            fp64_peak = float(json.load(f)["fp64_tflops"])
        fp64_kind = "measured (tools/fp64_peak on a B200 of this pool, profiles/r04_fp64_peak.json)"
    except Exception:
        pass
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        # the elasticity oracle (C, OpenMP over the host cores) on a bounded sample: the same
        # algorithm at 65^3 x 3 dofs, 5 levels (the 129^3 problem takes ~1 min per solve there)
        from oracle import oracle as O

        mg = O.ElastMG((65, 65, 65), nlevels - 1, smooth_its=m)
        bo = O.el_rhs((65, 65, 65))
        t1 = time.perf_counter()
        _, orep = mg.solve(bo, rtol=rtol)
        t_cpu = time.perf_counter() - t1
        cpu = {"value": bo.size / t_cpu, "unit": "DOF/s", "cores": int(os.environ.get("OMP_NUM_THREADS", os.cpu_count())),
               "kind": "port", "sample": f"elasticity oracle (oracle/tmg_elast_oracle.c, OpenMP) on 65^3 x 3 dofs, "
                                         f"{nlevels - 1} levels, V({m},{m}), rtol {rtol:g}: {orep['iterations']} its, "
                                         f"{t_cpu:.2f} s"}
    line = {
        "metric": "MG-CG DOF/s (time-to-solution)", "value": n_dof * args.steps / dev_t, "unit": "DOF/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_t / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded log-uniform element moduli, body force)",
        "config": {"workload": f"cfg5: {np3[0]}^3 Q1 elasticity x3 dof {nlevels}-level MG V({m},{m}) "
                               f"Cheb-point-block-Jacobi CG rtol {rtol:g}", "global_batch": 1,
                   "seq_len": np3[0], "parallelism": f"box{world}" + (f", telescope r={world} at L{stages[0][0]}"
                                                                      if stages else ""),
                   "iterations": its, "t_setup_s": t_setup,
                   "l2": "inputs larger than L2 (b, x 155 MB each)"},
        "e2e": {"value": n_dof * args.steps / e2e_t, "unit": "DOF/s", "h2d_bytes_per_step": 8 * n_dof,
                "d2h_bytes_per_step": 8 * n_dof},
        "gpu_launches": rep.kernel_launches * args.steps,
        "roofline": {"bound": "fp64", "achieved": fl / (ms * 1e-3) / 1e12, "peak": fp64_peak, "unit": "TFLOP/s",
                     "frac": fl / (ms * 1e-3) / 1e12 / fp64_peak, "traffic": None,
                     "peak_kind": fp64_kind,
                     "kernel": "k_el_apply (Q1 elasticity operator, fine level)", "ms_per_launch": ms,
                     "flops_per_launch": fl, "bytes_per_launch": by,
                     "hbm_GBs": by / (ms * 1e-3) / 1e9},
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="tmgx", choices=["tmgx", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--est", default="lanczos", choices=["lanczos", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--galerkin", choices=["on", "off"], default=None)
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("gloo", init_method="env://", world_size=world, rank=rank)

    if args.impl == "reference":
        run_reference(args, rank, world)
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return

    import ctypes

    import numpy as np
    import torch

    from paper_1604_07163_b200 import tmgx as T

    torch.cuda.set_device(local)
    np3, nlevels, m, kind, stages, rtol, scaling = resolve(args.config, world)
    tele_level = stages[0][0] if stages else None
    if kind == 2:
        run_elast(args, world, rank, local, np3, nlevels, m, rtol, stages, dist)
        return
    est = T.EST_LANCZOS if args.est == "lanczos" else T.EST_REFERENCE

    job = None
    if world > 1:  # node-local rendezvous name for the peer-memory transport
        obj = [T.job_token() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        job = obj[0]
    w = T.World(n_ranks=world, nproc=world, proc=rank, device=local, job=job)
    tele = [T.TelescopeStage(lv, r) for lv, r in stages]
    t0 = time.perf_counter()
    galerkin = GALERKIN.get(args.config, False) if args.galerkin is None else args.galerkin == "on"
    s = T.SolverNode(w, T.Problem(np3, kind, seed_k=SEED_K),
                     T.MGConfig(nlevels, m, est, telescope=tele, galerkin=galerkin))
    t_setup = time.perf_counter() - t0
    cfg = T.KrylovConfig("cg", rtol=rtol)
    cfg_e2e = T.KrylovConfig("cg", rtol=rtol, initial_guess_nonzero=False)  # x0 = 0: x is output only
    n_local = s.local_size()
    n_dof = np3[0] * np3[1] * np3[2]

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    def max_over_ranks(v):
        if not dist:
            return v
        t = torch.tensor([v], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident solves (value)
    for _ in range(max(args.warmup, 0)):
        rep = s.solve_seeded(SEED_F, cfg=cfg)
    barrier()
    launches = 0
    dev_times = []
    its = []
    with ClockSampler(local) as clk:
        t_wall0 = time.perf_counter()
        for _ in range(args.steps):
            rep = s.solve_seeded(SEED_F, cfg=cfg)
            dev_times.append(rep.t_solve_s)
            launches += rep.kernel_launches
            its.append(rep.iterations)
        barrier()
        t_wall = time.perf_counter() - t_wall0
    t_dev = max_over_ranks(sum(dev_times))
    value = n_dof * args.steps / t_dev

    # ---- end to end through the C-ABI with pinned host buffers (e2e)
    b_host = torch.empty(n_local, dtype=torch.float64, pin_memory=True)
    x_host = torch.zeros(n_local, dtype=torch.float64, pin_memory=True)
    b_np = s.rhs(SEED_F)
    b_host.numpy()[:] = b_np
    # x is output only (zero initial guess): it is not cleared between steps, since a CPU-side
    # clear leaves its cache lines dirty and slows the device's write-back of the result
    for _ in range(max(args.warmup, 1)):
        s.solve_ptr(b_host.data_ptr(), x_host.data_ptr(), False, cfg_e2e)
    barrier()
    e2e_t = 0.0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        rep_e = s.solve_ptr(b_host.data_ptr(), x_host.data_ptr(), False, cfg_e2e)
        e2e_t += time.perf_counter() - t0
    barrier()
    e2e_t = max_over_ranks(e2e_t)
    e2e = n_dof * args.steps / e2e_t

    # ---- roofline of the dominant kernel of the solve, live (CUDA events on the library stream)
    # The finest level runs the temporally blocked post-smooth (TMA-staged, 24 B/pt) when the
    # blocked smoother applies (m = 2, single-box level), else the fused Chebyshev pass.
    peak, peak_kind = read_peaks()
    tb = m in (2, 3) and world == 1 and os.environ.get("TMGX_TB", "1") != "0"
    if tb and m == 3:
        dom_id, dom_key, dom_name = (13, "tb3_post", "k_cheb3_tb<post> (blocked V(3,3) post-smooth, TMA-staged "
                                     "b, x~ and row planes, fine level)")
    elif tb:
        dom_id, dom_key, dom_name = (9, "tb_post", "k_cheb2_fast<post> (blocked V(2,2) post-smooth, TMA-staged, fine level)"
                                     if kind == 0 else "k_cheb2_tb<post> (blocked V(2,2) post-smooth, fine level)")
    else:
        dom_id, dom_key, dom_name = (1, "cheb_step_last", "k_cheb_step (last pass, fine level)")
    ms, by = s.bench_kernel(dom_id, nlevels - 1, iters=20)
    ms_all = max_over_ranks(ms)
    achieved = by / (ms_all * 1e-3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f).get(f"{args.config}:{dom_key}")
    except Exception:
        pass
    # every fine-level kernel of the path: live us/launch and algorithmic GB/s
    kernels = {}
    names = {1: "cheb_step_last", 3: "residual", 4: "restrict", 5: "prolong_add", 6: "cg_update", 7: "spmv_dot",
             8: "tb_pre", 9: "tb_post", 10: "prolong_to", 11: "resid_restrict", 12: "tb3_pre", 13: "tb3_post",
             15: "resid_restrict_sep"}
    if m == 3:
        names = {k: v for k, v in names.items() if k not in (8, 9)}
    else:
        names = {k: v for k, v in names.items() if k not in (12, 13)}
    for kid, kname in names.items():
        try:
            kms, kby = s.bench_kernel(kid, nlevels - 1, iters=10)
            kernels[kname] = {"us": round(kms * 1e3, 2), "GB/s": round(kby / (kms * 1e-3) / 1e9, 1)}
        except Exception:  # noqa: BLE001 (kernel not applicable to this level)
            pass

    # per-level V-cycle profile (device time per node, max over ranks; peer bytes, summed over
    # ranks): BASELINE configs[3] asks for per-level time and NVLink bytes
    levels = s.level_profile(reps=10)
    if dist:
        t = torch.tensor([lv["us"] for lv in levels], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        bsum = torch.tensor([float(lv["peer_bytes"]) for lv in levels], dtype=torch.float64)
        dist.all_reduce(bsum, op=dist.ReduceOp.SUM)
        for lv, u, by in zip(levels, t.tolist(), bsum.tolist()):
            lv["us"], lv["peer_bytes"] = u, int(by)
    for lv in levels:
        lv["us"] = round(lv["us"], 2)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, t_cpu, ckind, desc, _, _ = cpu_reference_sample(args.config, steps=1, warmup=0, galerkin=galerkin)
        cpu = {"value": rate, "unit": "DOF/s", "cores": 1, "kind": ckind, "sample": desc}

    if rank == 0:
        line = {
            "metric": "MG-CG DOF/s (time-to-solution)", "value": value, "unit": "DOF/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_dev / args.steps * 1e3,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded RHS, natural-index hash; BASELINE configs are synthetic)",
            "config": workload_config(args.config, world, tele_level, galerkin, args.est),
            "solve": {"iterations": its[-1] if its else None, "t_setup_s": t_setup,
                      "wall_ms_per_step": t_wall / args.steps * 1e3},
            "e2e": {"value": e2e, "unit": "DOF/s", "h2d_bytes_per_step": 8 * n_dof,
                    "d2h_bytes_per_step": 8 * n_dof},
            "gpu_launches": launches,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": dom_name, "peak_kind": peak_kind,
                         "bytes_per_launch": by, "ms_per_launch": ms_all, "fine_level_kernels": kernels,
                         "bytes_note": ("algorithmic bytes count the coefficient as 8 B/pt (k, SURVEY §8(d)); the "
                                        "var-coef kernels stream 4 precomputed row planes (32 B/pt)" if kind == 1
                                        else "algorithmic bytes (SURVEY §8(d))")},
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            "levels": levels,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
