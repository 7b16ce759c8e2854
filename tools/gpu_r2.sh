set -x
timeout 1200 python -m pytest tests/test_gpu_multiproc.py -q -x -rA 2>&1 | tail -30 > gpurun_out/r2_mp.log
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -8 > gpurun_out/r2_pytest.log
