"""Generate the golden fixtures from the reference (oracle/_ref, the unmodified reference
compiled with the FFTW-API stand-in). Run from the repo root:  python tests/golden/make_golden.py

schedules.json : RenderData of small graphs under every strategy (schedule.cpp:473-525)
renders.npz    : small renders — inputs, the reference's batched render() output
                 (render.cpp:14-81) and its per-node oracle output (reference.cpp:155-328)
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref  # noqa: E402


def graphs():
    out = []
    out.append(("chain_igo", np.array([0, 3, 1]), np.array([[0, 1, 0, 0], [1, 2, 0, 0]])))
    out.append(("parallel_eq", np.array([0, 0, 4, 4, 2, 1]),
                np.array([[0, 2, 0, 0], [1, 3, 0, 0], [2, 4, 0, 0], [3, 4, 0, 0], [4, 5, 0, 0]])))
    out.append(("parallel_edges_mix", np.array([0, 2, 1]), np.array([[0, 1, 0, 0], [0, 1, 0, 0], [1, 2, 0, 0]])))
    out.append(("one_by_one_quirk", np.array([0, 3, 2, 4, 4, 1]),
                np.array([[0, 1, 0, 0], [1, 2, 0, 0], [1, 2, 0, 0], [0, 3, 0, 0], [3, 4, 0, 0], [4, 2, 0, 0], [2, 5, 0, 0]])))
    t, e = ref.four_track_snippet()
    out.append(("fig1_snippet", t, e))
    t, e = ref.console(3)
    out.append(("console3", t, e))
    t, e = ref.console(16, 0.3, 16)
    out.append(("console16_p03_s16", t, e))
    for seed in (23, 24, 25, 26, 27):
        t, e = ref.random_dag(seed, 5, 40)
        out.append((f"random_dag_{seed}", t, e))
    return out


def schedules():
    cases = []
    for name, t, e in graphs():
        for strategy in (0, 1, 2, 3):
            if strategy == 3 and len(t) > 60:
                continue
            p = ref.Plan(t, e, strategy)
            cases.append({
                "name": name, "strategy": strategy, "types": [int(x) for x in t],
                "edges": [[int(v) for v in r] for r in np.asarray(e).reshape(-1, 4)],
                "type_codes": p.type_codes, "subsets": p.subsets, "sigma": p.sigma,
                "steps": [[s["type"], s["param_begin"], s["param_end"], s["store_begin"], s["store_end"], s["gather"],
                           s["aggregate"]] for s in p.steps],
                "param_source_rows": {str(k): v for k, v in p.param_source_rows.items()},
            })
    return cases


def renders():
    arrs = {}
    specs = [(13, 2000.0, 1024), (14, 2000.0, 1024), (15, 2000.0, 1024), (16, 2000.0, 1024)]
    for i, (seed, fs, n) in enumerate(specs):
        t, e = ref.random_dag(seed, 5, 25)
        params = ref.random_legal_params(t, e, seed)
        src = np.random.default_rng(seed).uniform(-1, 1, size=(int(np.sum(t == 0)), 1, 2, n))
        arrs[f"c{i}_types"], arrs[f"c{i}_edges"] = t, e
        arrs[f"c{i}_meta"] = np.array([fs, n], dtype=np.float64)
        for ty, m in params.items():
            arrs[f"c{i}_p{ty}"] = m
        arrs[f"c{i}_src"] = src
        arrs[f"c{i}_out"] = ref.Plan(t, e, 1).render(params, src, sample_rate=fs)
        arrs[f"c{i}_slow"] = ref.render_reference(t, e, params, src, sample_rate=fs)
    # A console with every processor type at 44.1 kHz.
    i = len(specs)
    t, e = ref.console(2, 0.0, 3)
    n = 4096
    params = ref.random_legal_params(t, e, 77)
    src = np.stack([ref.uniform_noise(2 * n, 1000 + k).reshape(1, 2, n) for k in range(int(np.sum(t == 0)))])
    arrs[f"c{i}_types"], arrs[f"c{i}_edges"] = t, e
    arrs[f"c{i}_meta"] = np.array([44100.0, n], dtype=np.float64)
    for ty, m in params.items():
        arrs[f"c{i}_p{ty}"] = m
    arrs[f"c{i}_src"] = src
    arrs[f"c{i}_out"] = ref.Plan(t, e, 1).render(params, src, sample_rate=44100.0)
    arrs["count"] = np.array([i + 1])
    return arrs


if __name__ == "__main__":
    with open(os.path.join(HERE, "schedules.json"), "w") as f:
        json.dump(schedules(), f, separators=(",", ":"))
    np.savez_compressed(os.path.join(HERE, "renders.npz"), **renders())
    print("wrote", os.listdir(HERE))
