#!/bin/bash
O=gpurun_out/${1:-s3v}
mkdir -p $O
for v in 0 5 6; do TMGX_PSPMV_MB=$v KB_TAG=mb_$v timeout 300 python tools/kbench.py cfg2 14 >> $O/kb.log 2>&1; TMGX_PSPMV_MB=$v python tools/ccprobe.py cfg2 >> $O/cc.log 2>&1; done
