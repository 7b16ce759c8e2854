#!/bin/bash
O=gpurun_out/${1:-v27}
mkdir -p $O
for v in 0 1 2 3; do TMGX_M27=$v KB_TAG=m27_$v timeout 300 python tools/kbench.py cfg3 0@6 1@6 3@6 >> $O/kb27.log 2>&1; done
for v in 0 1; do TMGX_VAR_K=$v KB_TAG=vark_$v timeout 300 python tools/kbench.py cfg3 1 3 7 >> $O/kbk.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -rf -k "golden or varcoef or apply or vcycle or galerkin" 2>&1 | tail -5 > $O/pytest.log
