#!/bin/bash
# ncu --set full of the config-5 union's FFT kernels (eq_conv, column passes, rows_conv_fk,
# cols_inv, reverb_ir) with their SASS source pages. Usage (GPU box): bash tools/c5_fft_profile.sh TAG
tag=${1:-fft}
export PYTHONPATH=.
ncu --set full --clock-control none --import-source on -k "regex:eq_conv|cols_fwd|rows_conv|cols_inv|reverb_ir" -c 8 -f \
    -o /tmp/${tag} python tools/c5_one_union.py --renders 1 > gpurun_out/${tag}.log 2>&1
ncu -i /tmp/${tag}.ncu-rep --page raw --csv | gzip > gpurun_out/${tag}_raw.csv.gz
for k in eq_conv rows_conv_fk cols_inv reverb_ir; do
  ncu -i /tmp/${tag}.ncu-rep --page source --csv --print-source sass -k regex:$k 2>/dev/null | gzip > gpurun_out/${tag}_src_$k.csv.gz
done
ncu -i /tmp/${tag}.ncu-rep --page source --csv --print-source sass -k "regex:cols_fwd<9, 1" 2>/dev/null | gzip > gpurun_out/${tag}_src_cols_fwd_sig.csv.gz
