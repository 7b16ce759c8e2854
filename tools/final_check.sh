#!/bin/bash
# Round-end style check on one B200: GPU tests, smoke, both bench arms (outputs: gpurun_out/final/).
O=gpurun_out/final
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -5 > $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench.log 2>&1
timeout 900 python bench.py --impl reference > $O/bench_ref.log 2>&1
