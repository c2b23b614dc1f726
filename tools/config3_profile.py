"""Config-3 diagnostics: per-step device time of one 64-console union (mg_profile_steps) and
the host-side costs of one batch (plan build, reorder, DeviceRenderer setup, enqueue).

Usage (GPU box): python tools/config3_profile.py [graphs] [seed]
"""
import os
import sys
import time

import numpy as np

import workloads as wl

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2408_03204_b200 as mg  # noqa: E402
from paper_2408_03204_b200 import sharding  # noqa: E402
from paper_2408_03204_b200.device import DeviceRenderer, profile_steps  # noqa: E402

L = 1 << 17


def main():
    graphs = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    st = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(st)
    t0 = time.perf_counter()
    members = [wl.generate_console_arrays(int(rng.integers(4, 33)), 0.3, 1000 * st + i) for i in range(graphs)]
    t, e = sharding.union_arrays(members)
    t1 = time.perf_counter()
    params = wl.random_legal_params(t, 5000 + st)
    t2 = time.perf_counter()
    rd = mg.compute_render_data_arrays(t, e)
    t3 = time.perf_counter()
    P = rd.reorder_params(params)
    t4 = time.perf_counter()
    procs = mg.ProcessorSet(sample_rate=44100.0, device=0)
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    dr = DeviceRenderer(rd, procs, 1, L, P, device=dev)
    torch.cuda.synchronize()
    t6 = time.perf_counter()
    dr.render()
    torch.cuda.synchronize()
    for _ in range(2):
        dr.render()
    torch.cuda.synchronize()
    t7 = time.perf_counter()
    dr.render()
    t8 = time.perf_counter()
    torch.cuda.synchronize()
    t9 = time.perf_counter()
    print(f"nodes {len(t)} edges {len(e)} steps {rd.num_steps} type_string {rd.schedule.type_codes()}")
    print(f"host ms: generate {1e3*(t1-t0):.1f} params {1e3*(t2-t1):.1f} plan {1e3*(t3-t2):.1f} "
          f"reorder {1e3*(t4-t3):.1f} DeviceRenderer {1e3*(t6-t5):.1f} enqueue {1e3*(t8-t7):.1f} render {1e3*(t9-t7):.1f}")
    ms = profile_steps(dr, reps=3)
    tot = float(ms.sum())
    for s, m in zip(rd.steps, ms):
        slots = s.store_end - s.store_begin
        print(f"  {mg.type_code(s.type)} slots {slots:5d} edges {len(s.gather):5d} {m*1e3:9.1f} us "
              f"{m*1e3/max(slots,1):7.2f} us/slot {100*m/tot:5.1f}%")
    print(f"sum of steps {tot:.2f} ms")


if __name__ == "__main__":
    main()
