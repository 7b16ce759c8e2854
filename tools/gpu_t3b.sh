#!/bin/bash
# m = 3 var-coef blocked kernel variants: kernel timings on cfg3, then the parity tests.
O=gpurun_out/${1:-t3b}
mkdir -p $O
timeout 300 python tools/kbench.py cfg3 12 13 1 3 7 > $O/kb_default.log 2>&1
TMGX_T3_NR=2 TMGX_T3_TY=8 KB_TAG=nr2ty8 timeout 300 python tools/kbench.py cfg3 12 13 > $O/kb_nr2.log 2>&1
TMGX_T3_LEAN=0 KB_TAG=generic timeout 300 python tools/kbench.py cfg3 12 13 > $O/kb_generic.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -rf -k "blocked_m3 or golden or varcoef or smoother or vcycle or apply" 2>&1 | tail -15 > $O/pytest_t3.log
timeout 900 python -m pytest tests/test_gpu_baseline_sizes.py -q -rf -k "cfg3" 2>&1 | tail -15 > $O/pytest_cfg3.log
timeout 900 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_cfg3.log 2>&1
