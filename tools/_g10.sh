timeout 900 python tools/telescope_table.py gpurun_out/telescope_table.csv > gpurun_out/g10_tele.log 2>&1
timeout 1500 python bench.py --config cfg3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/g10_cfg3.log 2>&1
