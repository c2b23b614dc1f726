"""Workload generators are bit-identical to the reference's; the C ABI library loads and
exports every symbol include/mixgraph_b200.h declares (no compute calls: CPU-safe)."""
import ctypes
import os
import re

import numpy as np

import workloads as wl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_header_symbols_exported(mg):
    hdr = open(os.path.join(ROOT, "include", "mixgraph_b200.h")).read()
    names = set(re.findall(r"\b(mg_[a-z0-9_]+)\s*\(", hdr))
    assert len(names) >= 30
    lib = ctypes.CDLL(mg.LIB_PATH)
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing


def test_param_widths_and_codes(mg):
    # types.cpp:14-25
    assert [mg.param_width(t) for t in range(10)] == [0, 0, 0, 2, 1024, 4, 4, 1, 768, 880]
    assert "".join(mg.type_code(t) for t in range(10)) == "iomgecnsrd"


def test_console_generator_matches_reference(mg, ref):
    for k in (1, 2, 5, 16, 32, 64):
        for prune, seed in ((0.0, 0), (0.3, 16), (0.7, 123)):
            t, e = ref.console(k, prune, seed)
            g = wl.generate_console(k, prune, seed)
            gt, ge = g.arrays()
            assert np.array_equal(gt, t) and np.array_equal(ge, e)
    assert mg.to_flat(wl.generate_console(8)).num_nodes() == 70  # 8K + 6


def test_random_legal_params_match_reference(mg, ref):
    for seed in range(6):
        t, e = ref.random_dag(seed, 10, 60)
        want = ref.random_legal_params(t, e, seed + 100)
        got = wl.random_legal_params(t, seed + 100)
        assert sorted(int(k) for k in got) == sorted(want)
        for k, v in want.items():
            assert np.array_equal(got[k], v)
    t, e = ref.console(16, 0.3, 16)
    want = ref.random_legal_params(t, e, 7)
    got = wl.random_legal_params(t, 7)
    for k, v in want.items():
        assert np.array_equal(got[k], v)


def test_uniform_noise_matches_reference(mg, ref):
    for seed in (0, 1, 1016):
        assert np.array_equal(mg.uniform_noise(5000, seed), ref.uniform_noise(5000, seed))


def test_default_params_and_checks(mg):
    d = mg.default_param_row(mg.NodeType.COMPRESSOR)
    assert list(d) == [0.995, -1.0, 0.5, 4.0]
    dl = mg.default_param_row(mg.NodeType.DELAY).reshape(40, 22)
    assert np.allclose(np.hypot(dl[:, 0], dl[:, 1]), 1.0, atol=1e-12)
    import pytest
    for bad in ([1.5, -1, 0.5, 4], [0.9, -1, -0.5, 4], [0.9, -1, 0.5, 0.5], [0.9, float("nan"), 0.5, 4]):
        with pytest.raises(ValueError):
            mg.check_param_row(mg.NodeType.COMPRESSOR, bad)
    row = np.zeros(880)
    row[0] = 1.2
    with pytest.raises(ValueError, match="unit disk"):
        mg.check_param_row(mg.NodeType.DELAY, row)


def test_knee_curves_continuous(mg):
    # test_processors.cpp:308-332 on the product's scalar curves
    rng = np.random.default_rng(23)
    for _ in range(500):
        T, W, R = rng.uniform(-10, 5), rng.uniform(1e-3, 5), rng.uniform(1, 20)
        top, bot = T + W, T - W
        assert abs(mg.compressor_gain_log(top, T, W, R) - (T + (top - T) / R)) <= 1e-9
        assert abs(mg.compressor_gain_log(bot, T, W, R) - bot) <= 1e-9
        assert abs(mg.noisegate_gain_log(top, T, W, R) - top) <= 1e-9
        assert abs(mg.noisegate_gain_log(bot, T, W, R) - (T + R * (bot - T))) <= 1e-9
