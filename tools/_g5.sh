timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/g5_pytest.log
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 1 > gpurun_out/g5_cfg5.log 2>&1
