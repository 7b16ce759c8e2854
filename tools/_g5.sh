timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/g5_pytest.log
timeout 600 python bench.py > gpurun_out/g5_bench.log 2>&1
