"""Forward/backward parity of long FFT convolutions (delay and reverb chains) against oracle/_ref
at lengths that cross the 2^20 .. 2^23 convolution sizes (test/diagnostic tool)."""
import sys
import numpy as np
import torch
from oracle import ref
import paper_2408_03204_b200 as mg

FS = 2000.0
for ty in (9, 8):
    for a in [int(x) for x in (sys.argv[1:] or ["19", "20", "21", "22"])]:
        g = mg.Graph(); g.add_serial_chain([0, ty, 1]); t, e = g.arrays()
        L = (1 << a) + 64
        rng = np.random.default_rng(a)
        src = rng.uniform(-1, 1, size=(1, 1, 2, L))
        params = ref.random_legal_params(t, e, a)
        procs = mg.ProcessorSet(sample_rate=FS)
        rd = mg.compute_render_data_arrays(t, e)
        dr = mg.DeviceRenderer(rd, procs, 1, L, rd.reorder_params(params))
        dr.sources.copy_(torch.as_tensor(src, dtype=torch.float32))
        out = dr.render().cpu().numpy()
        want = ref.Plan(t, e, 1).render(params, src, sample_rate=FS)
        err = ref.rel_linf(out, want)
        bad = np.nonzero(np.abs(out - want).max(axis=(0, 1, 2)) > 1e-3 * np.abs(want).max())[0]
        print(f"type {ty} L=2^{a}+64 rel_linf {err:.3e} first bad sample {bad[:1]} n_bad {bad.size}", flush=True)
