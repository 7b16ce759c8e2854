set -x
nvidia-smi --query-gpu=name,compute_mode --format=csv > gpurun_out/r1_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/r1_pytest.log
for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_parity.py -k "determinism or varcoef" -q 2>&1 | tail -3 >> gpurun_out/r1_det.log; done
timeout 600 python -m pytest tests/test_gpu_baseline_sizes.py -q -rA 2>&1 | tail -15 > gpurun_out/r1_big.log
