"""Per-node error in the first 64 samples vs the rest, for one config-3 member rendered inside
the union (DeviceRenderer arena) and alone (diagnostic). Usage: python tools/union_head_err.py STEP I"""
import sys

import numpy as np
import torch

import paper_2408_03204_b200 as mg
import workloads as wl
from oracle import ref
from paper_2408_03204_b200 import sharding

step, i = int(sys.argv[1]), int(sys.argv[2])
H = int(sys.argv[3]) if len(sys.argv) > 3 else 64
if len(sys.argv) > 4:
    mg.set_fft_precision(int(sys.argv[4]))
L = wl.L2
members = wl.config3_members(step)
t_u, e_u = sharding.union_arrays(members)
params = wl.random_legal_params(t_u, wl.config3_params_seed(step))
bank = wl.source_bank(64, L)
rd = mg.compute_render_data_arrays(t_u, e_u)
procs = mg.ProcessorSet()
offs = np.cumsum([0] + [int(np.sum(m[0] == 0)) for m in members])
noffs = np.cumsum([0] + [len(m[0]) for m in members])
dr = mg.DeviceRenderer(rd, procs, 1, L, rd.reorder_params(params))
dr.sources.copy_(torch.as_tensor(bank[[k % 64 for k in range(rd.num_inputs)]], dtype=torch.float32))
dr.render()
torch.cuda.synchronize()
sigma = np.asarray(rd.sigma)
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
want, winter = ref.Plan(t, e, 1).render(sl, src, keep_intermediates=True)
rd1 = mg.compute_render_data_arrays(t, e)
y1, i1 = mg.render(rd1, procs, rd1.reorder_params(sl), src, keep_intermediates=True)
rows = sigma[noffs[i]:noffs[i + 1]]
got = dr.arena.index_select(0, torch.as_tensor(rows, device=dr.arena.device)).cpu().numpy().astype(np.float64)
for n in range(len(t)):
    w = winter[n]
    print(f"{n:3d} {mg.type_name(int(t[n])):10s} head lvl {np.abs(w[..., :H]).max():.2e} union {np.abs(got[n][..., :H]-w[..., :H]).max():.2e} "
          f"alone {np.abs(i1[n][..., :H]-w[..., :H]).max():.2e} | tail lvl {np.abs(w[..., H:]).max():.2e} union {np.abs(got[n][..., H:]-w[..., H:]).max():.2e}")
