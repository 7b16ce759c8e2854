#!/bin/bash
O=gpurun_out/${1:-s3t}
mkdir -p $O
for v in 0 1; do TMGX_MARCH_PF2=$v KB_TAG=pf2_$v timeout 300 python tools/kbench.py cfg2 14 3 1 7 >> $O/kb_pf2.log 2>&1; done
for v in 0 1; do TMGX_MARCH_PF2=$v KB_TAG=pf2_$v timeout 300 python tools/kbench.py cfg3 14 3 1 >> $O/kb_pf2.log 2>&1; done
for v in 0 1; do TMGX_MARCH_PF2=$v python tools/ccprobe.py cfg2 >> $O/cc_pf2.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_acceptance.py tests/test_gpu_level_profile.py -q -rf 2>&1 | tail -12 > $O/pytest_acc.log
