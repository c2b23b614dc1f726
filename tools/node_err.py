"""Per-node relative error (vs the reference's intermediates) of config 2 under each FFT
precision. Usage: PYTHONPATH=. python tools/node_err.py"""
import numpy as np

import paper_2408_03204_b200 as mg
import workloads as wl
from oracle import ref

t, e, params = wl.config2()
L = wl.L2
src = wl.sources(int(np.sum(t == 0)), L)
want, winter = ref.Plan(t, e, 1).render(params, src, keep_intermediates=True)
procs = mg.ProcessorSet()
rd = mg.compute_render_data_arrays(t, e)
errs = {}
for bits in (32, 64):
    mg.set_fft_precision(bits)
    y, inter = mg.render(rd, procs, rd.reorder_params(params), src, keep_intermediates=True)
    errs[bits] = [np.abs(inter[n] - winter[n]).max() / max(np.abs(winter[n]).max(), 1e-300) for n in range(len(t))]
    print(bits, "out", ref.rel_linf(y, want))
for n in range(len(t)):
    print(n, mg.type_name(int(t[n])), f"{errs[32][n]:.2e} {errs[64][n]:.2e}")
