"""Per-node error of one config-3 member (product vs reference, intermediates in original
order) — diagnostic for the full-size parity tests. Usage: python tools/member_err.py STEP I"""
import sys

import numpy as np

import paper_2408_03204_b200 as mg
import workloads as wl
from oracle import ref
from paper_2408_03204_b200 import sharding

step, i = int(sys.argv[1]), int(sys.argv[2])
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
bank = wl.source_bank(64, wl.L2)
src = bank[[(offs[i] + j) % 64 for j in range(offs[i + 1] - offs[i])]]
rd = mg.compute_render_data_arrays(t, e)
procs = mg.ProcessorSet()
y, inter = mg.render(rd, procs, rd.reorder_params(sl), src, keep_intermediates=True)
want, winter = ref.Plan(t, e, 1).render(sl, src, keep_intermediates=True)
print("tracks", int(np.sum(t == 0)), "nodes", len(t), "out err", ref.rel_linf(y, want))
for n in range(len(t)):
    a, b = inter[n], winter[n]
    err = np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)
    print(n, mg.type_name(int(t[n])), f"peak {np.max(np.abs(b)):.3e} rel {err:.2e} abs {np.max(np.abs(a-b)):.2e}",
          "row", None if mg.param_width(int(t[n])) == 0 else sl[mg.NodeType(int(t[n]))][int(np.sum(t[:n] == t[n]))][:4])
