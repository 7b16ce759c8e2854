"""Builds the in-tree sm_100a shared libraries.

  libtmgx.so         performance build (nvcc may contract a*b+c into DFMA)
  libtmgx_parity.so  parity build (-fmad=false): V-cycle arithmetic bitwise equal to the CPU oracle

Both are plain nvcc invocations (no torch extension machinery); the .so files live next to
this file so they travel with the repository snapshot to the GPU box.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SOURCES = ["tmg_grid.cpp", "tmg_options.cpp", "tmgx_node.cpp", "tmgx_kernels.cu", "tmgx_engine.cu", "tmgx_elast.cu",
           "tmgx_capi.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def lib_path(parity=False):
    return os.path.join(HERE, "libtmgx_parity.so" if parity else "libtmgx.so")


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(parity=False, verbose=False, force=False):
    tag = "parity" if parity else "perf"
    objdir = os.path.join(HERE, "build", tag)
    os.makedirs(objdir, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".hpp", ".cuh", ".h"))]
    headers.append(os.path.join(ROOT, "include", "tmgx.h"))
    flags = ARCH + ["-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC,-ffp-contract=off",
                    "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-Xptxas", "-v"]
    if parity:
        flags += ["-fmad=false", "-DTMGX_PARITY"]
    flags += os.environ.get("TMGX_NVCC_EXTRA", "").split()  # tuning experiments (e.g. -DTMGX_TB_PF=6)
    # objects built with other flags (e.g. a TMGX_NVCC_EXTRA experiment) are never reused
    stamp = os.path.join(objdir, "flags.txt")
    if not os.path.exists(stamp) or open(stamp).read() != " ".join(flags):
        force = True
    cmds, objs = [], []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(objdir, src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            lang = ["-x", "cu"] if src.endswith(".cu") else []
            cmds.append(["nvcc"] + flags + lang + ["-c", s, "-o", o])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
        return r.stderr

    with ThreadPoolExecutor(max_workers=4) as ex:
        logs = list(ex.map(run, cmds))
    with open(stamp, "w") as f:
        f.write(" ".join(flags))
    if verbose:
        for lg in logs:
            sys.stdout.write(lg)
    out = lib_path(parity)
    if force or cmds or _stale(out, objs):
        run(["nvcc"] + ARCH + ["-shared", "-o", out] + objs + ["-lrt", "-cudart", "static"])
    return out


def build_all(verbose=False, force=False):
    with ThreadPoolExecutor(max_workers=2) as ex:  # the two builds in parallel
        fut = [ex.submit(build, p, verbose, force) for p in (False, True)]
        return [f.result() for f in fut]


if __name__ == "__main__":
    for p in build_all(verbose="-v" in sys.argv, force="-f" in sys.argv):
        print(p)
