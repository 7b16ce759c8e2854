timeout 300 python tools/tb_ab.py cfg2 >> gpurun_out/g5_ab.log 2>&1
TMGX_LIB=libtmgx_u3.so timeout 300 python tools/tb_ab.py cfg2 >> gpurun_out/g5_ab.log 2>&1
