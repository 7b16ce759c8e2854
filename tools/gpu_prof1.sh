# one-kernel A/B + ncu capture: bash tools/gpu_prof1.sh OUT KID [pytest -k expr]
O=gpurun_out/$1; K=$2
mkdir -p $O
if [ -n "$3" ]; then timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_sizes.py tests/test_gpu_determinism.py -k "$3" -q -rf 2>&1 | tail -8 > $O/pytest.log; fi
for k in 9 8; do timeout 300 python tools/profile_kernel.py $k >> $O/live.log 2>&1; TMGX_TB_FAST=0 timeout 300 python tools/profile_kernel.py $k >> $O/live_old.log 2>&1; done
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k_cheb2" -s 2 -c 1 -o $O/full python tools/profile_kernel.py $K > $O/full.log 2>&1
