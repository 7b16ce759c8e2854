timeout 900 python -m pytest tests -m gpu -x -q -k "elast" 2>&1 | tail -25 > gpurun_out/g5_pytest.log
