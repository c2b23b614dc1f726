"""Per-stream kernel timeline of one replayed config-2 render (CUPTI via torch.profiler's
chrome trace): start / duration / stream of every kernel. Usage:
PYTHONPATH=. python tools/render_timeline.py out.txt"""
import json
import sys
import tempfile

import torch
from torch.profiler import ProfilerActivity, profile

import paper_2408_03204_b200 as mg
import workloads as wl

t, e, params = wl.config2()
rd = mg.compute_render_data_arrays(t, e)
dr = mg.DeviceRenderer(rd, mg.ProcessorSet(), 1, wl.L2, rd.reorder_params(params))
dr.sources.copy_(torch.as_tensor(wl.sources(16, wl.L2), dtype=torch.float32))
g = dr.capture()
for _ in range(5):
    g.replay()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    g.replay()
    torch.cuda.synchronize()
path = tempfile.mktemp(suffix=".json")
prof.export_chrome_trace(path)
ev = [x for x in json.load(open(path))["traceEvents"] if x.get("cat") in ("kernel", "gpu_memset")]
t0 = min(x["ts"] for x in ev)
lines = []
for x in sorted(ev, key=lambda x: x["ts"]):
    name = x["name"].replace("mgb::", "").replace("(anonymous namespace)::", "").split("(")[0]
    lines.append(f"{x['ts'] - t0:8.1f} {x['dur']:7.1f}  stream {x['args'].get('stream', '?'):>4}  grid {str(x['args'].get('grid', '')):14s} {name[:60]}")
end = max(x["ts"] + x["dur"] for x in ev) - t0
lines.append(f"render span {end:.1f} us")
open(sys.argv[1], "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
