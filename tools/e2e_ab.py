import workloads as wl
"""e2e A/B of RenderPipeline double-audio conversion: host threads / host fraction vs device (config 2)."""
import os
import subprocess
import sys

for v in (sys.argv[1:] or ["0", "2", "4", "8"]):  # THREADS or THREADS:HOST_FRACTION
    t, _, f = v.partition(":")
    env = dict(os.environ, MGB_PIPELINE_HOST_THREADS=t, MGB_PIPELINE_HOST_FRACTION=f or "1")
    out = subprocess.run([sys.executable, "-c", """
import sys, time, json; sys.path.insert(0, '.')
import numpy as np, bench, paper_2408_03204_b200 as mg
g = wl.generate_console(16, 0.3, 16); fg = mg.to_flat(g); rd = mg.compute_render_data(fg)
P = rd.reorder_params(wl.random_legal_params(fg.node_types, 2024)); L = 1 << 17
src = np.stack([mg.uniform_noise(2 * L, 1000 + k).reshape(1, 2, L) for k in range(rd.num_inputs)])
procs = mg.ProcessorSet()
pipe = mg.RenderPipeline(rd, procs, 1, L, dtype=np.float64, depth=2)
ps = pipe.pinned(src.shape); ps[...] = src
outs = [pipe.pinned((1, 1, 2, L)) for _ in range(2)]
for i in range(5): pipe.submit(P, ps, outs[i % 2])
pipe.sync()
n = 40; t0 = time.perf_counter()
for i in range(n): pipe.submit(P, ps, outs[i % 2])
pipe.sync(); dt = (time.perf_counter() - t0) / n
want = mg.render(rd, procs, P, src)
print(json.dumps({'ms': dt * 1e3, 'nsps': 105 * L / dt, 'exact': bool(np.array_equal(outs[(n - 1) % 2], want))}))
"""], env=env, capture_output=True, text=True)
    print(v, out.stdout.strip(), out.stderr.strip()[-300:])
