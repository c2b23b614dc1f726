#!/bin/bash
# GPU-box profiling pass for one round (writes gpurun_out/; summarise with
# tools/ncu_render_summary.py). Each ncu command runs only after the same command exited 0
# without ncu. Usage: bash tools/profile_round.sh TAG
tag=${1:-rXX}
set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$tag.log 2>&1 || exit 1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_small_$tag.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_$tag.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_launches_$tag.log 2>&1
python tools/one_render.py --renders 2 > gpurun_out/one_render_$tag.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -c 58 -f -o gpurun_out/prof_render_$tag \
    python tools/one_render.py --renders 1 > gpurun_out/ncu_full_$tag.log 2>&1
ls -la gpurun_out/ | tail -12
tail -2 gpurun_out/ncu_full_$tag.log
