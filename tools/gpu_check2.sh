O=gpurun_out/s5b
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rf 2>&1 | tail -25 > $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py --config cfg5 --steps 10 --warmup 3 > $O/bench_cfg5.log 2>&1
