"""The EQ prologue's closed-form response basis (csrc/device/eq.cu: eq_basis_build) restated in
numpy and checked against the reference's own FIR design (`dsp.cpp:106-136`, zero_phase_fir via
oracle/_ref) followed by the 8192-point DFT the convolution uses. CPU only."""
import numpy as np
import pytest

from oracle import ref

FIR = 2047
NFFT = 8192
Q = 1024


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


def reference_response(log_mags):
    taps = np.zeros(FIR)
    lm = np.ascontiguousarray(log_mags, dtype=np.float64)
    assert ref.lib().ref_zero_phase_fir(lm.ctypes.data, FIR, taps.ctypes.data) == 0
    x = np.zeros(NFFT)
    c = (FIR - 1) // 2
    x[: c + 1] = taps[c:]
    x[NFFT - c:] = taps[:c]
    return np.real(np.fft.fft(x))[: NFFT // 2 + 1] / NFFT


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
