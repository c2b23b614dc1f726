#!/bin/bash
# ncu --set full of every kernel of one config-5 union render (first render after warm-up of
# the constants), raw page exported as CSV. Usage (GPU box): bash tools/c5_all_profile.sh TAG
tag=${1:-c5}
export PYTHONPATH=.
ncu --set full --clock-control none -f -o /tmp/${tag} python tools/c5_one_union.py --renders 1 > gpurun_out/${tag}_ncu.log 2>&1
ncu -i /tmp/${tag}.ncu-rep --page raw --csv | gzip > gpurun_out/${tag}_raw.csv.gz
