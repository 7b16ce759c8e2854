#!/bin/bash
O=gpurun_out/${1:-s3k}
mkdir -p $O
for v in 0 1; do TMGX_G27_SYM=$v KB_TAG=sym_$v timeout 300 python tools/kbench.py cfg3 0@6 1@6 3@6 >> $O/kb_sym.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_baseline_sizes.py -q -rf -k "cfg3" 2>&1 | tail -5 > $O/pytest_cfg3.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dropin.py -q -rf -k "galerkin or varcoef or golden or dropin or vcycle" 2>&1 | tail -8 > $O/pytest_g.log
timeout 900 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_cfg3.log 2>&1
