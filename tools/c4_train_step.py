"""One config-4 optimisation step (forward + MSE + backward + SGD) bracketed by
cudaProfilerStart/Stop after a warm-up step, for ncu --profile-from-start off."""
import os
import sys

import numpy as np

import workloads as wl

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2408_03204_b200 as mg  # noqa: E402
from paper_2408_03204_b200 import training  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 441000
t, e = wl.generate_large_console_arrays(64)
rd = mg.compute_render_data_arrays(t, e)
P = rd.reorder_params(wl.random_legal_params(t, 4040))
procs = mg.ProcessorSet()
tr = training.Trainer(rd, procs, 1, L, P, trainable=[int(x) for x in P], learning_rate=1e-3)
src = torch.rand((rd.num_inputs, 1, 2, L), device="cuda") * 2 - 1
tgt = torch.zeros((rd.buffer_rows - rd.output_begin, 1, 2, L), device="cuda")
tr.step(src, tgt)
torch.cuda.synchronize()
torch.cuda.profiler.start()
tr.step(src, tgt)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(3):
    tr.step(src, tgt)
b.record()
torch.cuda.synchronize()
print("ok", float(tr.loss.item()), "train step ms", a.elapsed_time(b) / 3)
