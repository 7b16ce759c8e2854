timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/g2_pytest.log
for cfg in "TMGX_TB=0" "TMGX_TB=1 TMGX_TB_ZC=16" "TMGX_TB=1 TMGX_TB_ZC=32" "TMGX_TB=1 TMGX_TB_ZC=64"; do
  env $cfg timeout 300 python tools/tb_ab.py cfg2 >> gpurun_out/g2_ab.log 2>&1
done
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/g2_bench.log 2>&1
