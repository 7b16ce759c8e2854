#!/bin/bash
O=gpurun_out/${1:-s3m}
mkdir -p $O
nproc > $O/nproc.txt; lscpu | head -20 >> $O/nproc.txt
timeout 600 python -m pytest tests/test_gpu_level_profile.py tests/test_capi_symbols.py -q -rf 2>&1 | tail -8 > $O/pytest_prof.log
timeout 900 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg4.log 2>&1
timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 > $O/bench_cfg5.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg2.log 2>&1
