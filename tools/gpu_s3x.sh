#!/bin/bash
O=gpurun_out/${1:-s3x}
mkdir -p $O
for v in 0 3 4; do TMGX_M27_SYM_MB=$v KB_TAG=symmb_$v timeout 300 python tools/kbench.py cfg3 0@6 1@6 3@6 >> $O/kb.log 2>&1; done
for v in 0 4 5; do TMGX_PSPMV_VAR_MB=$v KB_TAG=varmb_$v timeout 300 python tools/kbench.py cfg3 14 >> $O/kb.log 2>&1; done
