for r in 1 2; do
timeout 300 python tools/tb_ab.py cfg2 >> gpurun_out/g5_ab.log 2>&1
TMGX_LIB=libtmgx_wall.so timeout 300 python tools/tb_ab.py cfg2 >> gpurun_out/g5_ab.log 2>&1
done
timeout 300 python tools/tb_debug.py > gpurun_out/g5_debug.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "golden or vcycle or smoother" 2>&1 | tail -3 > gpurun_out/g5_pytest.log
