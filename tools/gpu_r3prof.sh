#!/bin/bash
# Round-3 (session) profile batch: default bench (cfg2, with the CPU reference beside it), the
# reference arm, cfg3 bench, cfg2 launch list, ncu full captures of the dominant kernels.
O=gpurun_out/${1:-r3prof}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 900 python bench.py > $O/bench_cfg2.log 2>&1
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_ref.log 2>&1
timeout 900 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_cfg3.log 2>&1
python tools/profile_solve.py --config cfg2 > $O/plain_solve.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file $O/launches_cfg2_solve.csv python tools/profile_solve.py --config cfg2 > $O/launches.log 2>&1
python tools/kbench.py cfg2 9 8 7 6 > $O/kb_cfg2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_cheb2_fast -c 2 -o $O/cfg2_tb python tools/kbench.py cfg2 9 8 > $O/ncu_tb.log 2>&1
python tools/kbench.py cfg3 12 13 > $O/kb_cfg3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_cheb3_var -c 2 -o $O/cfg3_tb3 python tools/kbench.py cfg3 12 13 > $O/ncu_tb3.log 2>&1
