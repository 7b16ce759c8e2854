timeout 300 python tools/tb_debug.py > gpurun_out/g3_debug.log 2>&1
TMGX_TB=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/g3_launches_tb0.csv python tools/profile_solve.py --config cfg2 > gpurun_out/g3_ncu.log 2>&1
