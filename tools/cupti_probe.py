"""Does torch.profiler (kineto / CUPTI) report the kernels inside a replayed render graph?"""
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2408_03204_b200 as mg
import workloads as wl

t, e, params = wl.config2()
L = wl.L2
rd = mg.compute_render_data_arrays(t, e)
procs = mg.ProcessorSet()
dr = mg.DeviceRenderer(rd, procs, 1, L, rd.reorder_params(params))
dr.sources.copy_(torch.as_tensor(wl.sources(16, L), dtype=torch.float32))
g = dr.capture()
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    g.replay()
    torch.cuda.synchronize()
ev = [x for x in prof.events() if x.device_type.name == "CUDA"]
print("cuda events", len(ev))
for x in sorted(ev, key=lambda x: x.time_range.start)[:40]:
    print(f"{x.time_range.start:12.1f} {x.time_range.end - x.time_range.start:8.2f} {x.name[:70]}")
