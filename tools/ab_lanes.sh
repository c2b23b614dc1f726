python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
for v in 0 1 0 1; do MGB_NO_LANES=$v python bench.py --steps 30 --warmup 5 > gpurun_out/bench_l$v.log 2>&1; echo "no_lanes=$v $(tail -1 gpurun_out/bench_l$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), d["steps_us"][1:3])')"; done
