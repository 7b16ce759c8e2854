O=gpurun_out/c2
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_sizes.py -k "smoother or vcycle or mgcg or cfg2 or estimator" -q -rf 2>&1 | tail -15 > $O/pytest.log
for f in 0 1; do TMGX_TB_FAST=$f timeout 300 python bench.py --no-cpu-baseline --steps 10 > $O/bench_fast$f.log 2>&1; done
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k_cheb2" -s 2 -c 1 -o $O/full_tb_post python tools/profile_kernel.py 9 > $O/full_tb_post.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k_cheb2" -s 2 -c 1 -o $O/full_tb_pre python tools/profile_kernel.py 8 > $O/full_tb_pre.log 2>&1
