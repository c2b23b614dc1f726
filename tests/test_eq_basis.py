"""The EQ prologue's two bases (csrc/device/eq.cu) restated in numpy and checked against the
reference's own FIR design (`dsp.cpp:106-136`, zero_phase_fir via oracle/_ref): the zero-phase
taps are linear in the magnitudes, h[c + t] = h[c - t] = sum_q exp(lm_q) D[q][t]
(eq_taps_basis_build, steps with many slots), and so is the 8192-bin response, R = A m with A
in closed form (eq_resp_basis_build, steps with few slots). CPU only."""
import numpy as np
import pytest

from oracle import ref

FIR = 2047
NFFT = 8192
Q = 1024
C = (FIR - 1) // 2


def _dirichlet(n, d):
    """D(2 pi n / d) with D(x) = sin(2047 x / 2) / sin(x / 2), exact-integer argument reduction."""
    n = np.mod(n, d)
    n = np.where(2 * n > d, n - d, n)
    m = np.mod(2047 * n, 2 * d)
    m = np.where(m > d, m - 2 * d, m)
    safe = np.where(n == 0, 1, n)
    v = np.sin(np.pi * m / d) / np.sin(np.pi * safe / d)
    return np.where(n == 0, 2047.0, v)


def _window_transform(n, d):
    s = d // 2046
    return 0.5 * _dirichlet(n, d) + 0.25 * _dirichlet(n + s, d) + 0.25 * _dirichlet(n - s, d)


def basis():
    """A[k][q] = response bin k (prescaled 1/8192) of the unit spectrum e_q, k <= 4096."""
    d = 2047 * 8192 * 2046
    k = np.arange(NFFT // 2 + 1, dtype=np.int64)[:, None]
    q = np.arange(Q, dtype=np.int64)[None, :]
    nq, nk = q * 8192 * 2046, k * 2047 * 2046
    cq = np.where(q == 0, 1.0, 2.0)
    return cq / (2.0 * 2047.0 * 8192.0) * (_window_transform(nq + nk, d) + _window_transform(nq - nk, d))


def design_basis():
    """D[q][t] = w(c + t) c_q cos(2 pi ((q t) mod 2047) / 2047) / 2047, t < 1024 (eq_taps_basis_build)."""
    q = np.arange(Q, dtype=np.int64)[:, None]
    t = np.arange(C + 1, dtype=np.int64)[None, :]
    w = 0.5 - 0.5 * np.cos(np.pi * 2.0 * (C + t) / (FIR - 1))
    cq = np.where(q == 0, 1.0, 2.0)
    return w * cq * np.cos(2.0 * np.pi * ((q * t) % FIR) / FIR) / FIR


def reference_taps(log_mags):
    taps = np.zeros(FIR)
    lm = np.ascontiguousarray(log_mags, dtype=np.float64)
    assert ref.lib().ref_zero_phase_fir(lm.ctypes.data, FIR, taps.ctypes.data) == 0
    return taps


def reference_response(log_mags):
    return response(reference_taps(log_mags))[: NFFT // 2 + 1]


def response(taps):
    x = np.zeros(NFFT)
    x[: C + 1] = taps[C:]
    x[NFFT - C:] = taps[:C]
    return np.real(np.fft.fft(x)) / NFFT


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
def test_design_basis_equals_reference_design():
    D = design_basis()
    rng = np.random.default_rng(7)
    for _ in range(3):
        lm = rng.uniform(-0.5, 0.5, Q)
        want = reference_taps(lm)
        half = np.exp(lm) @ D                      # h[c + t], t = 0..1023
        got = np.concatenate([half[:0:-1], half])  # h[c - t] mirrored
        assert np.max(np.abs(got - want)) <= 1e-12 * np.max(np.abs(want))
        assert np.max(np.abs(response(got) - response(want))) <= 1e-12 * np.max(np.abs(response(want)))
    # a flat spectrum (all log-mags 0) is the identity EQ: taps ~ a unit impulse at c
    flat = reference_taps(np.zeros(Q))
    half = np.ones(Q) @ D
    assert np.allclose(np.concatenate([half[:0:-1], half]), flat, rtol=0, atol=1e-15)


def test_basis_is_fp32_representable_scale():
    # every entry is a windowed cosine / 2047: |D| <= 2 / 2047, so fp32 rounding is ~1e-10 absolute
    D = design_basis()
    assert np.max(np.abs(D)) <= 2.0 / FIR + 1e-15


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
def test_closed_form_basis_equals_reference_design():
    A = basis()
    rng = np.random.default_rng(7)
    for _ in range(3):
        lm = rng.uniform(-0.5, 0.5, Q)
        want = reference_response(lm)
        got = A @ np.exp(lm)
        assert np.max(np.abs(got - want)) <= 1e-12 * np.max(np.abs(want))
    # a flat spectrum (all log-mags 0) is the identity EQ: response ~1/8192 on every bin
    flat = reference_response(np.zeros(Q))
    assert np.allclose(A @ np.ones(Q), flat, rtol=0, atol=1e-15)
