#!/bin/bash
O=gpurun_out/${1:-t3c}
mkdir -p $O
timeout 300 python tools/kbench.py cfg3 12 13 > $O/kb_default.log 2>&1
TMGX_T3_NR=2 TMGX_T3_TY=8 KB_TAG=nr2ty8 timeout 300 python tools/kbench.py cfg3 12 13 > $O/kb_nr2.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -rf -k "blocked_m3 or golden or varcoef" 2>&1 | tail -15 > $O/pytest_t3.log
timeout 900 python -m pytest tests/test_gpu_baseline_sizes.py -q -rf -k "cfg3" 2>&1 | tail -15 > $O/pytest_cfg3.log
timeout 900 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_cfg3.log 2>&1
python tools/kbench.py cfg3 13 > $O/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_cheb3_var -c 1 -o $O/t3post python tools/kbench.py cfg3 13 > $O/ncu.log 2>&1
