import workloads as wl
"""Same-box A/B timing of library builds: graph-replay ms/render of the config-2 workload.

Usage (GPU box):  python tools/ab_time.py ab/base.so ab/cur.so [...]
Each build runs in its own subprocess (MGB_LIB_OVERRIDE); builds are interleaved over
several rounds so clock/thermal drift hits all of them alike.
"""
import json
import os
import subprocess
import sys

CHILD = r"""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.environ["MGB_ROOT"])
import paper_2408_03204_b200 as mg
L = 1 << 17
g = wl.generate_console(16, 0.3, 16); fg = mg.to_flat(g); rd = mg.compute_render_data(fg)
P = rd.reorder_params(wl.random_legal_params(fg.node_types, 2024))
src = np.stack([mg.uniform_noise(2 * L, 1000 + k).reshape(1, 2, L) for k in range(rd.num_inputs)])
dr = mg.DeviceRenderer(rd, mg.ProcessorSet(), 1, L, P)
dr.sources.copy_(torch.as_tensor(src, dtype=torch.float32))
gr = dr.capture()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(5): gr.replay()
torch.cuda.synchronize()
ts = []
for _ in range(15):
    flush.fill_(1)
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): gr.replay()
    b.record(); b.synchronize()
    ts.append(a.elapsed_time(b) / 10)
print(json.dumps({"median_ms": float(np.median(ts)), "min_ms": float(np.min(ts))}))
"""


def main():
    libs = sys.argv[1:]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {l: [] for l in libs}
    for _ in range(3):
        for l in libs:
            env = dict(os.environ, MGB_LIB_OVERRIDE=os.path.abspath(l), MGB_ROOT=root)
            out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
            line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
            try:
                res[l].append(json.loads(line)["median_ms"])
            except Exception:
                print(l, "failed:", line)
    for l, v in res.items():
        print(f"{l:24s} median-of-medians {sorted(v)[len(v) // 2] if v else float('nan'):.4f} ms  runs {['%.4f' % x for x in v]}")


if __name__ == "__main__":
    main()
