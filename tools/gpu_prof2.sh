# A/B of the blocked smoother variants: bash tools/gpu_prof2.sh OUT [pytest -k expr]
O=gpurun_out/$1
mkdir -p $O
if [ -n "$2" ]; then TMGX_TBF_NR=4 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_sizes.py -k "$2" -q -rf 2>&1 | tail -8 > $O/pytest.log; fi
for k in 9 8; do
  for v in "TMGX_TB_FAST=0" "TMGX_TBF_NR=2" "TMGX_TBF_NR=4"; do echo -n "$v " >> $O/live.log; env $v timeout 300 python tools/profile_kernel.py $k >> $O/live.log 2>&1; done
done
TMGX_TBF_NR=4 timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k_cheb2" -s 2 -c 1 -o $O/full4 python tools/profile_kernel.py 9 > $O/full.log 2>&1
