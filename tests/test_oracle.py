"""The oracle itself: the compiled reference passes its own test-suite, and the FFTW-API
stand-in it links against restates FFTW's c2c contract (checked against numpy)."""
import ctypes
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = os.path.join(ROOT, "oracle", "_ref", "unit_tests")


@pytest.mark.skipif(not os.path.exists(UNIT), reason="oracle/_ref not built")
def test_reference_unit_tests_pass():
    r = subprocess.run([UNIT], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "test cases: 72 | passed: 72 | failed: 0" in r.stdout


def test_fftw_stand_in_matches_numpy(ref):
    lib = ctypes.CDLL(ref.REF_SO)
    lib.fftw_plan_dft_1d.restype = ctypes.c_void_p
    lib.fftw_plan_dft_1d.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_uint]
    lib.fftw_execute_dft.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    lib.fftw_destroy_plan.argtypes = [ctypes.c_void_p]
    rng = np.random.default_rng(0)
    for n in (1, 2, 7, 8, 39, 384, 2047, 4096, 6000, 1 << 17):
        for sign in (-1, 1):
            x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
            buf = np.ascontiguousarray(x.copy())
            p = lib.fftw_plan_dft_1d(n, buf.ctypes.data, buf.ctypes.data, sign, 0)
            lib.fftw_execute_dft(p, buf.ctypes.data, buf.ctypes.data)
            lib.fftw_destroy_plan(p)
            want = np.fft.fft(x) if sign < 0 else np.fft.ifft(x) * n
            assert np.max(np.abs(buf - want)) / np.max(np.abs(want)) < 1e-13, (n, sign)


def test_reference_known_answers(ref):
    # test_schedule.cpp:60-67 (Fig. 1 snippet) and the console type strings.
    t, e = ref.four_track_snippet()
    assert ref.Plan(t, e, 3).type_codes == "iecgmregro"
    t, e = ref.console(16, 0.3, 16)
    assert ref.Plan(t, e, 1).type_codes == "iecnsgrdmecsgo"
    assert ref.Plan(t, e, 2).type_codes == "iecnsgdrmecsgo"
    assert ref.Plan(t, e, 0).num_steps == 105


@pytest.mark.parametrize("tracks,seed,batch", [(4, 7, 1), (9, 3, 2)])
def test_parallel_oracle_render_equals_reference_render(ref, tracks, seed, batch):
    # ref_render_parallel (the full-size parity tests' oracle) is render.cpp's loop with each
    # step's slots on host threads: bit-identical outputs and intermediates.
    t, e = ref.console(tracks, 0.3, seed)
    params = ref.random_legal_params(t, e, 11)
    src = np.random.default_rng(seed).uniform(-1, 1, size=(int(np.sum(t == 0)), batch, 2, 3000))
    plan = ref.Plan(t, e, 1)
    want, inter = plan.render(params, src, sample_rate=8000.0, keep_intermediates=True)
    keep = [0, 3, 5, len(t) - 1]
    got, kept = plan.render_parallel(params, src, sample_rate=8000.0, threads=4, keep=keep)
    assert np.array_equal(got, want)
    assert np.array_equal(kept, inter[keep])
