"""Quick device-time check of the two headline workloads (A/B between builds):
config 2 (captured render, L2 flushed between iterations) and config 5 (512 graphs as 8
captured unions). Usage: PYTHONPATH=. python tools/perf_quick.py [c2] [c5] [dyn=0|1] [pair=0|1]"""
import json
import sys

import numpy as np
import torch

import bench
import paper_2408_03204_b200 as mg
import workloads as wl

what = [w for w in sys.argv[1:] if "=" not in w] or ["c2", "c5"]
for w in sys.argv[1:]:
    if w.startswith("dyn="):  # dyn=0: chained look-back scans only (A/B of the streaming scan)
        mg.set_dyn_stream(int(w[4:]))
    if w.startswith("pair="):  # pair=0: compressor -> noisegate as two streaming launches
        mg.set_dyn_pair(int(w[5:]))
dev = torch.device("cuda", 0)
procs = mg.ProcessorSet()
res = {}
if "c2" in what:
    c2 = bench.config2_lines(mg, procs, dev, steps=30)
    res["config2_ms"] = c2["ms_per_render"]
    res["config2_in_render_us"] = c2["in_render_us"]
if "c5" in what:
    graphs, mine, unions = bench.config5_shard(0, 1)
    bank = torch.as_tensor(wl.source_bank(64, wl.L2), dtype=torch.float32).to(dev)
    caps = []
    keep = []
    for idx in unions:
        t, rd, params = bench.union_case(mg, graphs, idx)
        dr = mg.DeviceRenderer(rd, procs, 1, wl.L2, rd.reorder_params(params), device=dev)
        dr.sources.copy_(bank[torch.arange(rd.num_inputs, device=dev) % 64])
        keep.append(dr)
        caps.append(dr.capture())

    def step():
        for g in caps:
            g.replay()

    for _ in range(3):
        step()
    ms = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        step()
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    res["config5_ms"] = float(np.median(ms))
print(json.dumps(res))
