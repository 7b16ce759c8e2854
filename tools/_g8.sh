timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/g8_launches.csv python tools/profile_solve.py --config cfg2 > gpurun_out/g8_ncu.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/g8_bench.log 2>&1
