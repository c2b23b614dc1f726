"""Where (in time) a config-3 union member's output error peaks (diagnostic).
Usage: python tools/union_member_err.py STEP I"""
import sys

import numpy as np
import torch

import paper_2408_03204_b200 as mg
import workloads as wl
from oracle import ref
from paper_2408_03204_b200 import sharding

step, i = int(sys.argv[1]), int(sys.argv[2])
L = wl.L2
members = wl.config3_members(step)
t_u, e_u = sharding.union_arrays(members)
params = wl.random_legal_params(t_u, wl.config3_params_seed(step))
bank = wl.source_bank(64, L)
rd = mg.compute_render_data_arrays(t_u, e_u)
procs = mg.ProcessorSet()
br = mg.BatchRenderer(procs, 1, L, mg.BatchRenderer.capacity_of(rd, procs, 1, L), depth=1)
out = torch.empty((rd.buffer_rows - rd.output_begin, 1, 2, L), dtype=torch.float32, pin_memory=True).numpy()
br.submit(rd, params, torch.as_tensor(bank, dtype=torch.float32).cuda(), out, validate=True)
br.sync()
offs = np.cumsum([0] + [int(np.sum(m[0] == 0)) for m in members])
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
src = bank[[(offs[i] + j) % 64 for j in range(offs[i + 1] - offs[i])]]
want = ref.Plan(t, e, 1).render(sl, src)[0, 0]
got = out[i, 0].astype(np.float64)
y1 = mg.render(mg.compute_render_data_arrays(t, e), procs, mg.compute_render_data_arrays(t, e).reorder_params(sl), src)[0, 0]
err = np.abs(got - want)
err1 = np.abs(y1 - want)
peak = np.abs(want).max()
print("union rel", err.max() / peak, "alone rel", err1.max() / peak, "peak", peak)
for lo, hi in [(0, 64), (64, 512), (512, 4096), (4096, 16384), (16384, 65536), (65536, L)]:
    print(f"[{lo},{hi}) level {np.abs(want[:, lo:hi]).max():.3e} union err {err[:, lo:hi].max():.3e} alone err {err1[:, lo:hi].max():.3e}")
n = int(np.argmax(err.max(axis=0)))
print("argmax", n, want[:, n], got[:, n])
