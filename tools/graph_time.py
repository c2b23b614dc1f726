"""Device time of the captured config-2 render (mean over reps, L2 flushed between), for
same-box A/B of environment switches: python tools/graph_time.py [reps]."""
import json
import os
import sys

import numpy as np

import workloads as wl

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2408_03204_b200 as mg  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
L = 1 << 17
g = wl.generate_console(16, 0.3, 16)
fg = mg.to_flat(g)
rd = mg.compute_render_data(fg)
P = rd.reorder_params(wl.random_legal_params(fg.node_types, 2024))
if "MGB_CONV_FUSE" in os.environ:  # A-B: -1 auto, 0 separate kernel-spectrum rows pass, 1 fused
    mg.set_conv_fuse(int(os.environ["MGB_CONV_FUSE"]))
procs = mg.ProcessorSet()
dr = mg.DeviceRenderer(rd, procs, 1, L, P)
dr.sources.copy_(torch.as_tensor(np.stack([mg.uniform_noise(2 * L, 1000 + k).reshape(1, 2, L)
                                           for k in range(rd.num_inputs)]), dtype=torch.float32))
gr = dr.capture()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
for _ in range(5):
    gr.replay()
ts = []
for i in range(reps):
    flush.fill_(i & 255)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    gr.replay()
    b.record(s)
    ts.append((a, b))
torch.cuda.synchronize()
ms = [a.elapsed_time(b) for a, b in ts]
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("MGB_")}, "mean_ms": float(np.mean(ms)),
                  "median_ms": float(np.median(ms)), "kernels": rd.kernel_count(1, L)}))
