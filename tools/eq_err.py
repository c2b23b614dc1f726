"""rel-Linf of the config-2 render (console-16, 2^17) and of a 16-EQ-node step vs the compiled
reference, for the current MGB_* environment (GPU box): python tools/eq_err.py"""
import json
import os
import sys

import numpy as np

import workloads as wl

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_03204_b200 as mg  # noqa: E402
from oracle import ref  # noqa: E402

L = 1 << 17
g = wl.generate_console(16, 0.3, 16)
fg = mg.to_flat(g)
rd = mg.compute_render_data(fg)
params = wl.random_legal_params(fg.node_types, 2024)
src = np.stack([mg.uniform_noise(2 * L, 1000 + k).reshape(1, 2, L) for k in range(rd.num_inputs)])
procs = mg.ProcessorSet()
out = mg.render(rd, procs, rd.reorder_params(params), src)
t, e = g.arrays()
want = ref.Plan(t, e, 1).render(params, src)
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("MGB_")},
                  "config2_rel_linf": float(ref.rel_linf(out, want))}))
