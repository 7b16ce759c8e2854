#!/bin/bash
# Round profile capture on one B200 (run under gpurun from the repo root):
#   launch list of one steady-state cfg2 solve, ncu --set full of the top fine-level kernels,
#   then the bench lines (both arms). Outputs under gpurun_out/prof/.
set -u
O=gpurun_out/prof
mkdir -p $O
timeout 600 python bench.py > $O/bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file $O/launches_cfg2_solve.csv python tools/profile_solve.py --config cfg2 > $O/launches.log 2>&1
for spec in "9:k_cheb2_tb:tb_post" "8:k_cheb2_tb:tb_pre" "6:k_cg_update:cg_update" "10:k_prolong_pair:prolong_to" \
            "3:FApply:residual" "4:k_restrict:restrict"; do
  IFS=: read kid kre name <<< "$spec"
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$kre" -s 2 -c 1 \
    -o $O/full_$name python tools/profile_kernel.py $kid > $O/full_$name.log 2>&1
done
