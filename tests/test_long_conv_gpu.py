"""GPU: long FFT convolutions (reverb, multitap delay) at any signal length.

The reference convolves any length with one next_pow2(L + taps - 1) transform
(`dsp.cpp:64-86`). The product uses segmented overlap-save (launch.hpp ConvGeom): a single
transform when it is the cheapest, else segments of 2^a points, so lengths past 2^22 render too.
Forward: against the reference renderer (oracle/_ref) across the old 2^20 limit, at
L + taps - 1 in {2^20 + 1, 2^21 + 64, 2^22 + 64} (fs = 2 kHz: 4000-tap kernels) and at 44.1 kHz
(88,200 taps), automatic and forced transform sizes (2^21 / 2^22-point transforms exercise the
2048-point row and column passes). Backward: the input gradient of a linear time-invariant
chain is the correlation of dL/dy with the kernel, which the REFERENCE computes exactly as the
time reversal of its own render of the reversed gradient; parameter gradients of the segmented
pass equal the single-transform pass and a central difference of the reference.
"""
import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]

TOL = 1e-4
REVERB, DELAY = 8, 9


def chain(mg, ty):
    g = mg.Graph()
    g.add_serial_chain([0, ty, 1])
    return g.arrays()


@pytest.fixture
def conv_log(mg):
    yield mg.set_conv_log
    mg.set_conv_log(0)


@pytest.fixture
def fp64(mg):
    mg.set_fft_precision(64)
    yield
    mg.set_fft_precision(32)


def device_render(mg, t, e, params, src, fs, backward=False):
    import torch
    procs = mg.ProcessorSet(sample_rate=fs)
    rd = mg.compute_render_data_arrays(t, e)
    k, b, _, n = src.shape
    dr = mg.DeviceRenderer(rd, procs, b, n, rd.reorder_params(params), backward=backward)
    dr.sources.copy_(torch.as_tensor(src, dtype=torch.float32))
    out = dr.render()
    return dr, rd, out


@pytest.mark.parametrize("ty", [DELAY, REVERB])
@pytest.mark.parametrize("fs,full,force", [
    (2000.0, (1 << 20) + 1, 0), (2000.0, (1 << 21) + 64, 0), (2000.0, (1 << 22) + 64, 0),
    (2000.0, (1 << 21) + 64, 21), (2000.0, (1 << 21) + 64, 22), (2000.0, (1 << 22) + 64, 22),
    (44100.0, (1 << 21) + 88199, 0), (44100.0, (1 << 20) + 1, 0)])
def test_long_forward_matches_reference(mg, ref, conv_log, ty, fs, full, force):
    taps = int(round(2 * fs))
    L = full - taps + 1
    t, e = chain(mg, ty)
    params = ref.random_legal_params(t, e, 7 + ty)
    src = np.random.default_rng(full % 1000).uniform(-1, 1, size=(1, 1, 2, L))
    conv_log(force)
    _, _, out = device_render(mg, t, e, params, src, fs)
    want = ref.Plan(t, e, 1).render(params, src, sample_rate=fs)
    err = ref.rel_linf(out.cpu().numpy(), want)
    assert err < TOL, (L, err)


def test_batched_long_delay_segments(mg, ref):
    # batch 2: segments of both batch items (item = (slot*batch + b)*nseg + j) land in their rows
    fs, L = 2000.0, (1 << 20) + 5000
    t, e = chain(mg, DELAY)
    params = ref.random_legal_params(t, e, 3)
    src = np.random.default_rng(3).uniform(-1, 1, size=(1, 2, 2, L))
    _, _, out = device_render(mg, t, e, params, src, fs)
    want = ref.Plan(t, e, 1).render(params, src, sample_rate=fs)
    assert ref.rel_linf(out.cpu().numpy(), want) < TOL


@pytest.mark.parametrize("ty", [DELAY, REVERB])
@pytest.mark.parametrize("fs,full", [(2000.0, (1 << 20) + 1), (2000.0, (1 << 22) + 64), (44100.0, (1 << 21) + 88199)])
def test_long_input_gradient_matches_reference_correlation(mg, ref, ty, fs, full):
    import torch
    taps = int(round(2 * fs))
    L = full - taps + 1
    t, e = chain(mg, ty)
    params = ref.random_legal_params(t, e, 11 + ty)
    rng = np.random.default_rng(full % 997)
    src = rng.uniform(-1, 1, size=(1, 1, 2, L))
    w = rng.uniform(-1, 1, size=(1, 1, 2, L))
    dr, rd, out = device_render(mg, t, e, params, src, fs, backward=True)
    _, gsrc = dr.backward(torch.as_tensor(w, dtype=torch.float32, device=out.device))
    got = gsrc.cpu().numpy()
    # dL/dx[m] = sum_k h[k] w[m + k] = rev(h * rev(w))[m]: the reference's own causal convolution
    want = ref.Plan(t, e, 1).render(params, np.ascontiguousarray(w[..., ::-1]), sample_rate=fs)[..., ::-1]
    assert ref.rel_linf(got, want) < TOL


@pytest.mark.parametrize("ty", [DELAY, REVERB])
def test_long_param_gradients_segmented_equal_single(mg, ref, conv_log, ty):
    import torch
    fs = 2000.0
    L = (1 << 21) + 64 - 3999
    t, e = chain(mg, ty)
    params = ref.random_legal_params(t, e, 5 + ty)
    rng = np.random.default_rng(ty)
    src = rng.uniform(-1, 1, size=(1, 1, 2, L))
    w = rng.uniform(-1, 1, size=(1, 1, 2, L))
    grads = []
    for force in (0, 22):  # automatic: 2^15-point segments; 22: one 2^22 transform
        conv_log(force)
        dr, rd, out = device_render(mg, t, e, params, src, fs, backward=True)
        g, _ = dr.backward(torch.as_tensor(w, dtype=torch.float32, device=out.device))
        torch.cuda.synchronize()
        grads.append(g[ty].cpu().numpy())
    scale = np.abs(grads[1]).max()
    assert np.abs(grads[0] - grads[1]).max() <= 2e-3 * scale
    if ty == DELAY:
        # central differences of the reference on two active tap magnitudes
        tab = params[ty].reshape(-1, 22)
        picks = [r * 22 + 2 + m for r in range(tab.shape[0]) for m in (0, 5) if tab[r, 2:].max() > -60][:2]
        flat = params[ty].reshape(-1)
        plan = ref.Plan(t, e, 1)
        for i in picks:
            h = 1e-5
            hi = {k: np.array(v, copy=True) for k, v in params.items()}
            lo = {k: np.array(v, copy=True) for k, v in params.items()}
            hi[ty].reshape(-1)[i] += h
            lo[ty].reshape(-1)[i] -= h
            fd = (np.sum(w * plan.render(hi, src, sample_rate=fs)) - np.sum(w * plan.render(lo, src, sample_rate=fs))) / (2 * h)
            assert abs(grads[0].reshape(-1)[i] - fd) <= 2e-3 * max(abs(fd), scale), (i, grads[0].reshape(-1)[i], fd)
        assert flat.size == grads[0].size


@pytest.mark.parametrize("ty", [DELAY, REVERB])
def test_fp64_transforms_long_forward_and_gradient(mg, ref, fp64, ty):
    # mg_set_fft_precision(64): the same segmented convolution with fp64 arithmetic (fp32 arena)
    # matches the reference, forward and input gradient, across several segments.
    import torch
    fs, L = 2000.0, (1 << 20) + 3000
    t, e = chain(mg, ty)
    params = ref.random_legal_params(t, e, 21 + ty)
    rng = np.random.default_rng(ty + 40)
    src = rng.uniform(-1, 1, size=(1, 1, 2, L))
    w = rng.uniform(-1, 1, size=(1, 1, 2, L))
    dr, rd, out = device_render(mg, t, e, params, src, fs, backward=True)
    plan = ref.Plan(t, e, 1)
    assert ref.rel_linf(out.cpu().numpy(), plan.render(params, src, sample_rate=fs)) < 2e-6
    _, gsrc = dr.backward(torch.as_tensor(w, dtype=torch.float32, device=out.device))
    want = plan.render(params, np.ascontiguousarray(w[..., ::-1]), sample_rate=fs)[..., ::-1]
    assert ref.rel_linf(gsrc.cpu().numpy(), want) < 2e-6
