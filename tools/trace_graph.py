"""Kernel timeline of one captured config-2 render (torch.profiler / CUPTI), warm L2.

Usage (GPU box):  python tools/trace_graph.py [--no-graph]
Prints each kernel's start offset, duration and stream within one render, plus the
critical-path view: main-stream busy time vs. gaps.
"""
import argparse
import os
import sys

if "--serial" in sys.argv:  # every prologue inline on the main stream: isolated kernel times
    os.environ["MGB_NO_HOIST"] = "1"

import numpy as np

import workloads as wl
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2408_03204_b200 as mg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--serial", action="store_true")
    ap.add_argument("--length", type=int, default=1 << 17)
    args = ap.parse_args()
    L = args.length
    g = wl.generate_console(16, 0.3, 16)
    fg = mg.to_flat(g)
    rd = mg.compute_render_data(fg)
    P = rd.reorder_params(wl.random_legal_params(fg.node_types, 2024))
    src = np.stack([mg.uniform_noise(2 * L, 1000 + k).reshape(1, 2, L) for k in range(rd.num_inputs)])
    procs = mg.ProcessorSet()
    dr = mg.DeviceRenderer(rd, procs, 1, L, P)
    dr.sources.copy_(torch.as_tensor(src, dtype=torch.float32))
    run = dr.render if args.no_graph else dr.capture().replay
    for _ in range(5):
        run()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            run()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA" and e.time_range.elapsed_us() > 0]
    evs.sort(key=lambda e: e.time_range.start)
    # the 3 renders launch the same kernels: report the last third
    n = len(evs) // 3
    groups = [evs[i * n:(i + 1) * n] for i in range(3)]
    last = groups[-1]
    t0 = last[0].time_range.start
    end = max(e.time_range.end for e in last)
    print(f"renders seen: {len(groups)}; last render span {end - t0:.1f} us, {len(last)} kernels")
    for e in last:
        name = e.name.replace("void ", "").replace("mgb::(anonymous namespace)::", "")[:60]
        print(f"{e.time_range.start - t0:8.1f} {e.time_range.elapsed_us():8.1f} {e.time_range.end - t0:8.1f}  {name}")


if __name__ == "__main__":
    main()
