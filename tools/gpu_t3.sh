#!/bin/bash
# m = 3 blocked smoother: parity tests, cfg3 solve parity at size, cfg3 bench.
O=gpurun_out/${1:-t3}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -rf -k "blocked_m3 or golden or varcoef or smoother" 2>&1 | tail -15 > $O/pytest_t3.log
timeout 900 python -m pytest tests/test_gpu_baseline_sizes.py -q -rf -k "cfg3" 2>&1 | tail -15 > $O/pytest_cfg3.log
timeout 900 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_cfg3.log 2>&1
