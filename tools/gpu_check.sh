#!/bin/bash
# One-B200 check: GPU tests, smoke, bench (cfg2, cfg3), launch list of the cfg2 bench.
O=gpurun_out/${1:-chk}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf 2>&1 | tail -25 > $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > $O/bench.log 2>&1
timeout 900 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_cfg3.log 2>&1
