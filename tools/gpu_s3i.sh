#!/bin/bash
O=gpurun_out/${1:-s3i}
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_dropin.py -q -rf 2>&1 | tail -15 > $O/pytest_dropin.log
oracle/_ref/tmg_ref_gpupc 65 5 3 1 1 42 > $O/dropin_65.json 2>&1
for t in 0 1; do TMGX_T3_TREE=$t KB_TAG=tree_$t timeout 300 python tools/kbench.py cfg3 12 13 >> $O/kb_tree.log 2>&1; done
timeout 1500 python -m pytest tests -m gpu -q -rf 2>&1 | tail -15 > $O/pytest_all.log
