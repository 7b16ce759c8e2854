for v in mb4 pf2mb5; do TMGX_LIB=libtmgx_$v.so timeout 300 python tools/tb_ab.py cfg2 >> gpurun_out/g5_ab.log 2>&1; done
