#!/bin/bash
O=gpurun_out/${1:-s3q}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_sizes.py -q -rf -k "elast or cfg5" 2>&1 | tail -6 > $O/pytest_el.log
timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg5.log 2>&1
