timeout 300 compute-sanitizer --tool racecheck python tools/tb_debug9.py > gpurun_out/g4_race.log 2>&1
timeout 300 compute-sanitizer --tool synccheck python tools/tb_debug9.py > gpurun_out/g4_sync.log 2>&1
timeout 300 compute-sanitizer --tool initcheck python tools/tb_debug9.py > gpurun_out/g4_init.log 2>&1
timeout 300 compute-sanitizer --tool memcheck python tools/tb_debug9.py > gpurun_out/g4_mem.log 2>&1
