#!/bin/bash
# Round-end style check on one B200: GPU suite, smoke, bench lines (cfg2 default with the CPU
# reference beside it, the reference arm, cfg3, cfg4, cfg5), clocks.
O=gpurun_out/${1:-final}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rf 2>&1 | tail -25 > $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench_cfg2.log 2>&1
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > $O/bench_ref.log 2>&1
timeout 900 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_cfg3.log 2>&1
timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 > $O/bench_cfg5.log 2>&1
