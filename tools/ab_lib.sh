#!/bin/bash
# A/B of two builds of libmgb200.so on one box (GPU): the in-tree build vs gpurun_ab_base.so
# (copy of a baseline build at the repo root). Usage: bash tools/ab_lib.sh c5|c2
export PYTHONPATH=.
L=paper_2408_03204_b200/libmgb200.so
cp $L /tmp/new.so
for i in 1 2 3; do
  cp /tmp/new.so $L; echo -n "new "; python tools/perf_quick.py ${1:-c5} 2>&1 | tail -1
  cp gpurun_ab_base.so $L; echo -n "base "; python tools/perf_quick.py ${1:-c5} 2>&1 | tail -1
done
cp /tmp/new.so $L
