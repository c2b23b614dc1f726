"""A/B of the FFT-step arithmetic precision (32 vs 64 bits) on config 2: device time per
render (captured graph, L2 flushed), per-step times, and error vs the reference.
Usage: PYTHONPATH=. python tools/precision_ab.py"""
import json

import numpy as np
import torch

import paper_2408_03204_b200 as mg
import workloads as wl
from oracle import ref
from paper_2408_03204_b200.device import profile_steps

t, e, params = wl.config2()
L = wl.L2
src = wl.sources(int(np.sum(t == 0)), L)
want = ref.Plan(t, e, 1).render(params, src)
procs = mg.ProcessorSet()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
res = {}
for bits in (32, 64, 32, 64):
    mg.set_fft_precision(bits)
    rd = mg.compute_render_data_arrays(t, e)
    dr = mg.DeviceRenderer(rd, procs, 1, L, rd.reorder_params(params))
    dr.sources.copy_(torch.as_tensor(src, dtype=torch.float32))
    g = dr.capture()
    for _ in range(3):
        g.replay()
    ms = []
    for i in range(20):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    out = dr.outputs.cpu().numpy()
    steps = profile_steps(dr, reps=10)
    res[bits] = {"ms_median": float(np.median(ms)), "rel_linf": ref.rel_linf(out, want),
                 "steps_us": [[mg.type_code(s.type), round(float(x) * 1e3, 1)] for s, x in zip(rd.steps, steps)]}
    print(bits, json.dumps(res[bits]), flush=True)
