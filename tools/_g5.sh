timeout 300 python tools/tb_ab.py cfg2 >> gpurun_out/g5_ab.log 2>&1
TMGX_FUSE_DOTS=0 timeout 300 python tools/tb_ab.py cfg2 >> gpurun_out/g5_ab.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "golden or vcycle or options" 2>&1 | tail -3 > gpurun_out/g5_pytest.log
