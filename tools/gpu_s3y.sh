#!/bin/bash
O=gpurun_out/${1:-s3y}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_baseline_sizes.py -q -rf -k "fused or cfg3" 2>&1 | tail -5 > $O/pytest.log
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > $O/bench_ref.log 2>&1
timeout 1200 python tools/mp_levels.py cfg4 8 > $O/mp_cfg4_8.json 2> $O/mp_cfg4_8.err
timeout 900 python tools/mp_levels.py cfg2 4 > $O/mp_cfg2_4.json 2> $O/mp_cfg2_4.err
timeout 1200 python tools/mp_levels.py cfg3 8 > $O/mp_cfg3_8.json 2> $O/mp_cfg3_8.err
