# parity subset under one env + A/B live timings: bash tools/gpu_abt.sh OUT "PYTEST_ENV" "ENV1" "ENV2" ...
O=gpurun_out/$1; PE=$2; shift 2
mkdir -p $O
env $PE timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_sizes.py tests/test_gpu_determinism.py -k "smoother or vcycle or mgcg or cfg2 or repeat" -q -rf 2>&1 | tail -8 > $O/pytest.log
for k in 9 8; do for v in "$@"; do echo -n "$v " >> $O/live.log; env $v timeout 300 python tools/profile_kernel.py $k >> $O/live.log 2>&1; done; done
