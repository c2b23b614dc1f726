#!/bin/bash
# ncu --set full of the config-5 union's delay_cols and cols_inv with their SASS source pages.
# Usage (GPU box): bash tools/c5_cols_profile.sh TAG
tag=${1:-cols}
export PYTHONPATH=.
ncu --set full --clock-control none --import-source on -k "regex:delay_cols|cols_inv" -c 3 -f \
    -o /tmp/${tag} python tools/c5_one_union.py --renders 1 > gpurun_out/${tag}.log 2>&1
ncu -i /tmp/${tag}.ncu-rep --page raw --csv | gzip > gpurun_out/${tag}_raw.csv.gz
for k in delay_cols cols_inv; do
  ncu -i /tmp/${tag}.ncu-rep --page source --csv --print-source sass -k regex:$k 2>/dev/null | gzip > gpurun_out/${tag}_src_$k.csv.gz
done
