"""Minimal config-2 workload for profilers: ProcessorSet + DeviceRenderer, then `--renders`
eager renders (default 2) on the default stream. Used by tools/profile_round.sh under ncu."""
import argparse
import os
import sys

import numpy as np

import workloads as wl
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_03204_b200 as mg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--renders", type=int, default=2)
    ap.add_argument("--length", type=int, default=1 << 17)
    args = ap.parse_args()
    L = args.length
    fg = mg.to_flat(wl.generate_console(16, 0.3, 16))
    rd = mg.compute_render_data(fg)
    P = rd.reorder_params(wl.random_legal_params(fg.node_types, 2024))
    src = np.stack([mg.uniform_noise(2 * L, 1000 + k).reshape(1, 2, L) for k in range(rd.num_inputs)])
    dr = mg.DeviceRenderer(rd, mg.ProcessorSet(), 1, L, P)
    dr.sources.copy_(torch.as_tensor(src, dtype=torch.float32))
    for _ in range(args.renders):
        dr.render()
    torch.cuda.synchronize()
    print("ok", float(dr.outputs.abs().max()))


if __name__ == "__main__":
    main()
