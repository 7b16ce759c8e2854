#!/bin/bash
O=gpurun_out/${1:-el}
mkdir -p $O
python tools/el_solve.py > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launches_cfg5.csv python tools/el_solve.py > $O/l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_el_apply -c 1 --profile-from-start off -o $O/el_apply python tools/el_solve.py > $O/ncu.log 2>&1
