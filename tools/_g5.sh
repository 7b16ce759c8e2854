for t in 0 100 200; do TMGX_TB_MIN=$t timeout 300 python tools/tb_ab.py cfg2 >> gpurun_out/g5_ab.log 2>&1; done
for t in 0 100 200; do TMGX_TB_MIN=$t timeout 300 python tools/tb_ab.py cfg2 >> gpurun_out/g5_ab.log 2>&1; done
