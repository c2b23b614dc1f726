"""One config-3 render (a 64-console union) bracketed by cudaProfilerStart/Stop, for ncu
--profile-from-start off (per-kernel metrics of a large-grid render). Usage: python
tools/c3_one_render.py [graphs] [seed]"""
import os
import sys

import numpy as np

import workloads as wl

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2408_03204_b200 as mg  # noqa: E402
from paper_2408_03204_b200 import sharding  # noqa: E402

L = 1 << 17
graphs = int(sys.argv[1]) if len(sys.argv) > 1 else 64
st = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rng = np.random.default_rng(st)
members = [wl.generate_console_arrays(int(rng.integers(4, 33)), 0.3, 1000 * st + i) for i in range(graphs)]
t, e = sharding.union_arrays(members)
rd = mg.compute_render_data_arrays(t, e)
procs = mg.ProcessorSet(sample_rate=44100.0, device=0)
dr = mg.DeviceRenderer(rd, procs, 1, L, rd.reorder_params(wl.random_legal_params(t, 5000 + st)))
bank = torch.as_tensor(np.stack([mg.uniform_noise(2 * L, 1000 + k).reshape(1, 2, L) for k in range(64)]),
                       dtype=torch.float32).cuda()
dr.sources.copy_(bank[torch.arange(rd.num_inputs, device="cuda") % 64])
dr.render()
torch.cuda.synchronize()
torch.cuda.profiler.start()
dr.render()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok", len(t), rd.schedule.type_codes())
