"""GPU: the reverse-mode pass (parameter and source gradients) against central differences.

The reference has no autodiff (`SPEC.md:14`); its only gradient is the central difference of
`fit.cpp:70-82`, so that is the oracle here — taken on the REFERENCE's own double-precision
renderer (oracle/_ref), which makes the finite differences accurate to ~1e-8 while the
device pass computes in fp32. Loss L = sum(w * outputs) with fixed random weights w, so
dL/d(outputs) = w. Tolerance: |analytic - FD| <= 2e-3 * max(|FD| over the sampled entries,
|analytic| over the whole table) per parameter type (fp32 arithmetic through long FFT
correlations and scans: the error is absolute at the scale of the type's largest gradient).
"""
import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]

FS = 2000.0
TOL = 2e-3


def chain(mg, types):
    g = mg.Graph()
    g.add_serial_chain([0] + list(types) + [1])
    return g.arrays()


def analytic(mg, t, e, params, src, w, **cfg):
    import torch
    procs = mg.ProcessorSet(sample_rate=FS, **cfg)
    rd = mg.compute_render_data_arrays(t, e)
    k, b, _, n = src.shape
    dr = mg.DeviceRenderer(rd, procs, b, n, rd.reorder_params(params), backward=True)
    dr.sources.copy_(torch.as_tensor(src, dtype=torch.float32))
    out = dr.render().clone()
    grads, gsrc = dr.backward(torch.as_tensor(w, dtype=torch.float32, device=out.device))
    torch.cuda.synchronize()
    g = rd.original_order({t_: v.cpu().numpy() for t_, v in grads.items()})
    return out.cpu().numpy(), g, gsrc.cpu().numpy()


def fd_loss(ref, t, e, params, src, w, **cfg):
    y = ref.Plan(t, e, 1).render(params, src, sample_rate=FS, **cfg)
    return float(np.sum(w * y))


def check_params(mg, ref, t, e, params, src, w, picks=6, seed=0, skip=None, **cfg):
    out, g, _ = analytic(mg, t, e, params, src, w, **cfg)
    rng = np.random.default_rng(seed)
    for ty, tab in params.items():
        tab = np.asarray(tab)
        flat = tab.reshape(-1)
        idx = rng.choice(flat.size, size=min(picks, flat.size), replace=False)
        if ty == mg.NodeType.DELAY:  # magnitudes of active taps (positions: gradient 0, checked below)
            cols = np.arange(flat.size) % 22
            active = [i for i in range(flat.size) if cols[i] >= 2 and tab.reshape(-1, 22)[i // 22, 2:].max() > -60]
            idx = rng.choice(active, size=min(picks, len(active)), replace=False)
            pos = [i for i in range(flat.size) if cols[i] < 2]
            assert np.all(g[ty].reshape(-1)[pos] == 0.0)
        got, want = [], []
        for i in idx:
            h = 1e-5 * max(1.0, abs(flat[i]))
            hi = {k: np.array(v, copy=True) for k, v in params.items()}
            lo = {k: np.array(v, copy=True) for k, v in params.items()}
            hi[ty].reshape(-1)[i] += h
            lo[ty].reshape(-1)[i] -= h
            want.append((fd_loss(ref, t, e, hi, src, w, **cfg) - fd_loss(ref, t, e, lo, src, w, **cfg)) / (2 * h))
            got.append(g[ty].reshape(-1)[i])
        got, want = np.array(got), np.array(want)
        # fp32 FFT correlations carry an absolute error relative to the type's largest
        # gradient, so entries are judged against max(|FD| of the picks, max |grad| of the type).
        scale = max(np.abs(want).max(), np.abs(g[ty]).max(), 1e-12)
        assert np.abs(got - want).max() <= TOL * scale, (mg.type_name(ty), got, want)
    return out


@pytest.mark.parametrize("types", [[3], [7], [4], [5], [6], [8], [9], [3, 4, 5, 7]])
def test_chain_param_grads_match_central_differences(mg, ref, types):
    t, e = chain(mg, types)
    rng = np.random.default_rng(len(types) * 10 + types[0])
    L = 3000
    src = rng.uniform(-1, 1, size=(1, 1, 2, L))
    w = rng.uniform(-1, 1, size=(1, 1, 2, L))
    params = ref.random_legal_params(t, e, 7 + types[0])
    check_params(mg, ref, t, e, params, src, w, seed=types[0])


@pytest.mark.parametrize("gate", [False, True])
def test_dynamics_truncated_envelope_grads(mg, ref, gate):
    # envelope_taps < L: the FIR truncation term a^Ne e[n-Ne] is active in both passes.
    t, e = chain(mg, [6 if gate else 5])
    rng = np.random.default_rng(3)
    L = 2999
    src = rng.uniform(-1, 1, size=(1, 2, 2, L))
    w = rng.uniform(-1, 1, size=(1, 2, 2, L))
    params = ref.random_legal_params(t, e, 11)
    params[6 if gate else 5][0, 0] = 0.97  # a^Ne well above the 1e-30 cut
    check_params(mg, ref, t, e, params, src, w, picks=4, envelope_taps=300)


def test_console_param_and_source_grads(mg, ref):
    t, e = ref.console(2, 0.0, 5)
    rng = np.random.default_rng(5)
    L = 2500
    k = int(np.sum(t == 0))
    src = rng.uniform(-1, 1, size=(k, 1, 2, L))
    w = rng.uniform(-1, 1, size=(1, 1, 2, L))
    params = ref.random_legal_params(t, e, 21)
    out = check_params(mg, ref, t, e, params, src, w, picks=3, seed=2)
    want = ref.Plan(t, e, 1).render(params, src, sample_rate=FS)
    assert ref.rel_linf(out, want) < 1e-4
    # source gradient at a few samples
    _, _, gsrc = analytic(mg, t, e, params, src, w)
    for (kk, c, n) in [(0, 0, 10), (1, 1, 1200), (0, 1, 2499)]:
        h = 1e-4
        a, b = src.copy(), src.copy()
        a[kk, 0, c, n] += h
        b[kk, 0, c, n] -= h
        fd = (fd_loss(ref, t, e, params, a, w) - fd_loss(ref, t, e, params, b, w)) / (2 * h)
        assert abs(gsrc[kk, 0, c, n] - fd) <= 2e-3 * max(1.0, abs(fd)), (kk, c, n, gsrc[kk, 0, c, n], fd)


def test_backward_is_deterministic(mg, ref):
    t, e = ref.console(3, 0.3, 8)
    rng = np.random.default_rng(8)
    L = 4096
    src = rng.uniform(-1, 1, size=(int(np.sum(t == 0)), 2, 2, L))
    w = rng.uniform(-1, 1, size=(1, 2, 2, L))
    params = ref.random_legal_params(t, e, 9)
    _, g1, s1 = analytic(mg, t, e, params, src, w)
    _, g2, s2 = analytic(mg, t, e, params, src, w)
    assert np.array_equal(s1, s2)
    for ty in g1:
        assert np.array_equal(g1[ty], g2[ty])


@pytest.mark.parametrize("trainable,lr,ptol", [([3, 7], 0.5, 2e-3), ([5, 6], 2e-6, 1e-2)])
def test_fit_matches_reference_fit(mg, ref, trainable, lr, ptol):
    # fit.cpp:25-96 takes central differences (fd_step 1e-3) and descends; the analytic
    # gradients must follow the same trajectory. Dynamics: a small rate keeps the reference's
    # alpha +- fd_step probes inside (0, 1), and its fd_step = 1e-3 difference of a^k sums is
    # itself ~0.5% off the derivative in alpha, hence the looser parameter tolerance.
    from paper_2408_03204_b200 import training
    t, e = ref.console(1, 0.0, 2)
    rng = np.random.default_rng(12)
    L = 1500
    src = rng.uniform(-1, 1, size=(1, 1, 2, L))
    params = ref.random_legal_params(t, e, 13)
    for ty in (5, 6):
        params[ty][:, 0] = np.minimum(params[ty][:, 0], 0.99)
    target = ref.Plan(t, e, 1).render(ref.random_legal_params(t, e, 14), src, sample_rate=FS)
    want_p, want_h = ref.fit(t, e, params, src, target, trainable, 3, lr, sample_rate=FS)
    procs = mg.ProcessorSet(sample_rate=FS)
    fg = mg.to_flat(mg.Graph.from_arrays(t, e))
    got_p, got_h = training.fit(fg, params, procs, src, target, trainable=trainable, steps=3, learning_rate=lr)
    assert np.all(np.diff(want_h) < 0)
    assert np.allclose(got_h, want_h, rtol=2e-3, atol=0), (got_h, want_h)
    for ty in trainable:
        moved = np.abs(want_p[ty] - params[ty]).max()
        assert moved > 0
        assert np.abs(got_p[ty] - want_p[ty]).max() <= ptol * moved + 1e-12, (ty, got_p[ty], want_p[ty])
    for ty in params:
        if int(ty) not in trainable:
            assert np.array_equal(got_p[ty], params[ty])
