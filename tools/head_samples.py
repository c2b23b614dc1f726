"""Sample-level view of the bus compressor's first samples of one config-3 member rendered
alone (product vs reference): input l, r, mid = l + r, output. Diagnostic.
Usage: PYTHONPATH=. python tools/head_samples.py STEP I"""
import sys

import numpy as np

import paper_2408_03204_b200 as mg
import workloads as wl
from oracle import ref
from paper_2408_03204_b200 import sharding

step, i = int(sys.argv[1]), int(sys.argv[2])
L = wl.L2
members = wl.config3_members(step)
t_u, _ = sharding.union_arrays(members)
params = wl.random_legal_params(t_u, wl.config3_params_seed(step))
sl, off = {}, {}
for j, (t, _) in enumerate(members):
    for ty, tab in params.items():
        n = int(np.sum(t == int(ty)))
        if n:
            o = off.get(ty, 0)
            if j == i:
                sl[ty] = np.ascontiguousarray(tab[o:o + n])
            off[ty] = o + n
t, e = members[i]
offs = np.cumsum([0] + [int(np.sum(m[0] == 0)) for m in members])
bank = wl.source_bank(64, L)
src = bank[[(offs[i] + j) % 64 for j in range(offs[i + 1] - offs[i])]]
rd = mg.compute_render_data_arrays(t, e)
procs = mg.ProcessorSet()
y, inter = mg.render(rd, procs, rd.reorder_params(sl), src, keep_intermediates=True)
want, winter = ref.Plan(t, e, 1).render(sl, src, keep_intermediates=True)
comp = [n for n in range(len(t)) if t[n] == 5][-1]  # bus compressor: last compressor node
eq = comp - 1
print("bus compressor row", sl[mg.NodeType.COMPRESSOR][-1])
for n in range(12):
    ul, ur = winter[eq][0, 0, n], winter[eq][0, 1, n]
    pl, pr = inter[eq][0, 0, n], inter[eq][0, 1, n]
    print(f"n={n:2d} ref u=({ul:+.6e},{ur:+.6e}) mid {ul + ur:+.6e} | prod mid {pl + pr:+.6e} dmid {pl + pr - ul - ur:+.2e}"
          f" | out ref {winter[comp][0, 0, n]:+.6e} prod {inter[comp][0, 0, n]:+.6e}")
