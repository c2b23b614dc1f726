"""Error distribution of config-3 / config-5 union members against the reference, alongside the
error of the reference's own arithmetic over an fp32 arena (rows rounded to float between
steps: the floor any fp32-storage renderer faces). Diagnostic. Usage:
python tools/parity_survey.py [c3 STEPS...] [c5]"""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

import paper_2408_03204_b200 as mg
import workloads as wl
from oracle import ref
from paper_2408_03204_b200 import sharding

L = wl.L2
bank = wl.source_bank(64, L)
bank_dev = torch.as_tensor(bank, dtype=torch.float32).cuda()
procs = mg.ProcessorSet()


def union_case(members, params, per):
    t_u, e_u = sharding.union_arrays(members)
    rd = mg.compute_render_data_arrays(t_u, e_u)
    br = mg.BatchRenderer(procs, 1, L, mg.BatchRenderer.capacity_of(rd, procs, 1, L), depth=1)
    out = torch.empty((rd.buffer_rows - rd.output_begin, 1, 2, L), dtype=torch.float32, pin_memory=True).numpy()
    br.submit(rd, params, bank_dev, out, validate=True)
    br.sync()
    offs = np.cumsum([0] + [int(np.sum(m[0] == 0)) for m in members])

    def one(i):
        t, e = members[i]
        src = bank[[(offs[i] + j) % 64 for j in range(offs[i + 1] - offs[i])]]
        p = ref.Plan(t, e, 1)
        w = p.render_parallel(per[i], src, threads=1)
        w32 = p.render_parallel(per[i], src, threads=1, perturb=1e-6)
        pk = np.abs(w).max()
        return np.abs(out[i] - w[0]).max() / pk, np.abs(w32 - w).max() / pk

    with ThreadPoolExecutor(os.cpu_count()) as pool:
        return list(pool.map(one, range(len(members))))


def slices(members, params):
    out, off = [], {}
    for t, _ in members:
        p = {}
        for ty, tab in params.items():
            n = int(np.sum(t == int(ty)))
            if n:
                o = off.get(ty, 0)
                p[ty] = np.ascontiguousarray(tab[o:o + n])
                off[ty] = o + n
        out.append(p)
    return out


res = []
args = sys.argv[1:] or ["c3", "0", "1", "2", "c5"]
if args[0].startswith("fp"):
    mg.set_fft_precision(int(args[0][2:]))
    args = args[1:]
mode = None
for a in args:
    if a in ("c3", "c5"):
        mode = a
        if a == "c5":
            graphs = wl.config5_graphs()
            for shard in sharding.lpt_shards([sharding.graph_cost(t, L) for t, _ in graphs], 8)[:2]:
                members = [graphs[i] for i in shard]
                per = [wl.config5_member_params(i, graphs[i][0]) for i in shard]
                r = union_case(members, wl.union_params([t for t, _ in members], per), per)
                res += [("c5", k, x, y) for k, (x, y) in enumerate(r)]
        continue
    st = int(a)
    members = wl.config3_members(st)
    t_u, _ = sharding.union_arrays(members)
    params = wl.random_legal_params(t_u, wl.config3_params_seed(st))
    r = union_case(members, params, slices(members, params))
    res += [(f"c3/{st}", k, x, y) for k, (x, y) in enumerate(r)]
e = np.array([x for _, _, x, _ in res])
f = np.array([y for _, _, _, y in res])
print(f"members {len(res)}  product max {e.max():.3e} p99 {np.quantile(e, .99):.3e} median {np.median(e):.3e}")
print(f"global-noise probe (1e-6): max {f.max():.3e} p99 {np.quantile(f, .99):.3e} median {np.median(f):.3e}")
print(f"ratio product / probe: max {np.max(e / f):.2f} median {np.median(e / f):.2f}")
for c, k, x, y in sorted(res, key=lambda r: -r[2])[:10]:
    print(c, k, f"product {x:.3e} probe {y:.3e}")
