#!/bin/bash
# ncu --set full of the config-5 union's dynamics kernels: streaming scan (default) and the
# chained look-back scan (dyn=0). Usage (GPU box): bash tools/c5_dyn_profile.sh TAG
tag=${1:-dyn}
export PYTHONPATH=.
ncu --set full --clock-control none --import-source on -k regex:dyn_ -c 3 -f -o /tmp/${tag}_stream python tools/c5_one_union.py --renders 1 > gpurun_out/${tag}_stream.log 2>&1
ncu -i /tmp/${tag}_stream.ncu-rep --page raw --csv | gzip > gpurun_out/${tag}_stream_raw.csv.gz
ncu -i /tmp/${tag}_stream.ncu-rep --page source --csv -k regex:dyn_stream 2>/dev/null | gzip > gpurun_out/${tag}_stream_src.csv.gz
ncu --set full --clock-control none --import-source on -k regex:dyn_ -c 3 -f -o /tmp/${tag}_chain python tools/c5_one_union.py --renders 1 --dyn 0 > gpurun_out/${tag}_chain.log 2>&1
ncu -i /tmp/${tag}_chain.ncu-rep --page raw --csv | gzip > gpurun_out/${tag}_chain_raw.csv.gz
