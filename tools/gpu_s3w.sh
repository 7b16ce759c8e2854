#!/bin/bash
O=gpurun_out/${1:-s3w}
mkdir -p $O
KB_TAG=$2 timeout 300 python tools/kbench.py cfg2 14 3 1 7 >> $O/kb.log 2>&1
KB_TAG=$2 timeout 300 python tools/kbench.py cfg3 14 3 >> $O/kb.log 2>&1
python tools/ccprobe.py cfg2 >> $O/cc.log 2>&1
python tools/ccprobe.py cfg3 >> $O/cc.log 2>&1
