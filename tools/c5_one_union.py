"""One render of config-5 union `--union` (default 0) through DeviceRenderer, uncaptured (ncu
target for the conv / EQ / scan kernels at config-5 scale). Usage:
  PYTHONPATH=. python tools/c5_one_union.py [--union 0] [--renders 1]"""
import argparse

import torch

import bench
import paper_2408_03204_b200 as mg
import workloads as wl

ap = argparse.ArgumentParser()
ap.add_argument("--union", type=int, default=0)
ap.add_argument("--renders", type=int, default=1)
ap.add_argument("--dyn", type=int, default=-1, help="mg_set_dyn_stream mode (0: chained scans)")
args = ap.parse_args()
mg.set_dyn_stream(args.dyn)
dev = torch.device("cuda", 0)
procs = mg.ProcessorSet()
graphs, mine, unions = bench.config5_shard(0, 1)
t, rd, params = bench.union_case(mg, graphs, unions[args.union])
bank = torch.as_tensor(wl.source_bank(64, wl.L2), dtype=torch.float32).to(dev)
dr = mg.DeviceRenderer(rd, procs, 1, wl.L2, rd.reorder_params(params), device=dev)
dr.sources.copy_(bank[torch.arange(rd.num_inputs, device=dev) % 64])
for _ in range(args.renders):
    dr.render()
torch.cuda.synchronize()
print("ok", len(t), "nodes")
