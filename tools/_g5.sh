for v in p4 p6 p8; do TMGX_LIB=libtmgx_$v.so timeout 300 python tools/tb_ab.py cfg2 >> gpurun_out/g5_ab.log 2>&1; done
