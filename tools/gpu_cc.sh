#!/bin/bash
O=gpurun_out/${1:-cc}
mkdir -p $O
python tools/ccprobe.py cfg2 >> $O/cc.log 2>&1
for c in 9 17 33; do for cl in 8 16; do TMGX_CC_MAX=$c TMGX_CC_CLUSTER=$cl python tools/ccprobe.py cfg2 >> $O/cc.log 2>&1; done; done
TMGX_GRAPHS=0 python tools/ccprobe.py cfg2 >> $O/cc.log 2>&1
