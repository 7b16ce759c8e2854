timeout 300 python tools/tb_debug.py > gpurun_out/g5_debug.log 2>&1
timeout 300 python tools/tb_ab.py cfg2 >> gpurun_out/g5_ab.log 2>&1
TMGX_FUSE_RR=0 timeout 300 python tools/tb_ab.py cfg2 >> gpurun_out/g5_ab.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "transfer or vcycle or golden" 2>&1 | tail -15 > gpurun_out/g5_pytest.log
