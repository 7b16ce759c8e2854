#!/bin/bash
# cfg3: launch list of a 5-iteration solve, full capture of the Galerkin 27-point Chebyshev step.
O=gpurun_out/${1:-p3}
mkdir -p $O
python tools/profile_solve.py --config cfg3 --max-its 5 > $O/plain_solve.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file $O/launches_cfg3_solve.csv python tools/profile_solve.py --config cfg3 --max-its 5 > $O/launches.log 2>&1
python tools/kbench.py cfg3 0@6 1@6 3@6 > $O/kb27.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_march27 -c 1 -o $O/m27step python tools/kbench.py cfg3 0@6 > $O/ncu27.log 2>&1
