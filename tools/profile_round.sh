#!/bin/bash
# GPU-box profiling pass for one round (writes gpurun_out/; summarise with
# tools/ncu_render_summary.py gpurun_out/raw_TAG.csv.gz profiles/TAG). Each ncu command runs
# only after the same command exited 0 without ncu. The full report stays in /tmp on the box
# (gpurun brings back at most 64 MiB); its raw page and source pages come back as CSV.
tag=${1:-rXX}
set -x
nproc > gpurun_out/host_$tag.txt; lscpu >> gpurun_out/host_$tag.txt 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$tag.log 2>&1 || exit 1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_small_$tag.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_$tag.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_launches_$tag.log 2>&1
python tools/one_render.py --renders 2 > gpurun_out/one_render_$tag.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -c 58 -f -o /tmp/prof_render_$tag \
    python tools/one_render.py --renders 1 > gpurun_out/ncu_full_$tag.log 2>&1
ncu -i /tmp/prof_render_$tag.ncu-rep --page raw --csv | gzip > gpurun_out/raw_$tag.csv.gz
python tools/ncu_render_summary.py gpurun_out/raw_$tag.csv.gz gpurun_out/$tag > gpurun_out/summary_$tag.log 2>&1
python tools/ncu_stalls.py gpurun_out/raw_$tag.csv.gz > gpurun_out/stalls_$tag.txt 2>&1
ls -la gpurun_out/ | tail -16
tail -2 gpurun_out/ncu_full_$tag.log
