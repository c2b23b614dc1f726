"""GPU parity: the CUDA render path (through the C ABI) against the compiled reference.

Tolerance (north star): rel-L-inf = max|a-b| / max|b| <= 1e-4 against the reference's
double-precision output (`tests/support/test_util.cpp:126-135`), fp32 device arithmetic.
Cases follow `proj/tests/test_render.cpp` and `test_processors.cpp`, plus full-size
BASELINE configurations checked directly against the reference renderer.
"""
import numpy as np

import workloads as wl
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]

TOL = 1e-4
N = None


@pytest.fixture(scope="module")
def procs_small(mg):
    return mg.ProcessorSet(sample_rate=2000.0)


def rel(a, b):
    from oracle.ref import rel_linf
    return rel_linf(a, b)


def make(mg, t, e):
    return mg.to_flat(mg.Graph.from_arrays(t, e))


def render_both(mg, ref, t, e, params, src, fs, strategy=1, procs=None, **cfg):
    fg = make(mg, t, e)
    rd = mg.compute_render_data(fg, strategy)
    procs = procs or mg.ProcessorSet(sample_rate=fs, **cfg)
    got = mg.render(rd, procs, rd.reorder_params(params), src)
    want = ref.Plan(t, e, strategy).render(params, src, sample_rate=fs, **cfg)
    return got, want


# ---- processors -----------------------------------------------------------------------------

@pytest.mark.parametrize("t", [2, 3, 7, 4, 5, 6, 8, 9])
@pytest.mark.parametrize("fs,length", [(1000.0, 600), (44100.0, 8192), (44100.0, 5001)])
def test_processor_matches_reference(mg, ref, t, fs, length):
    rng = np.random.default_rng(t * 31 + length)
    slots, batch = 3, 2
    params = None
    if mg.param_width(t):
        g = mg.Graph()
        for _ in range(slots):
            g.add_node(t)
        gt, ge = g.arrays()
        params = ref.random_legal_params(gt, ge, 43 + t)[t]
    x = rng.uniform(-1, 1, size=(slots, batch, 2, length))
    procs = mg.ProcessorSet(sample_rate=fs)
    got = procs.process(t, x, slots, batch, length, params, 0)
    want = ref.process(t, x, slots, batch, length, params, 0, sample_rate=fs)
    for s in range(slots):
        assert rel(got[s], want[s]) < TOL, (t, s)


def test_gain_and_imager_known_answers(mg):
    procs = mg.ProcessorSet()
    rng = np.random.default_rng(3)
    u = rng.uniform(-1, 1, size=(2, 2, 500))
    u32 = u.astype(np.float32).astype(np.float64)
    assert np.array_equal(procs.process_node(mg.NodeType.GAIN, u, [0.0, 0.0]), u32)
    ones = np.ones((1, 2, 100))
    y = procs.process_node(mg.NodeType.GAIN, ones, [np.log(2.0), 0.0])
    assert abs(y[0, 0, 50] - 2.0) < 1e-6 and abs(y[0, 1, 50] - 1.0) < 1e-6
    hard = np.zeros((1, 2, 64))
    hard[0, 0] = 1.0
    y = procs.process_node(mg.NodeType.IMAGER, hard, [np.log(0.5)])
    assert abs(y[0, 0, 10] - 0.75) < 1e-6 and abs(y[0, 1, 10] - 0.25) < 1e-6


def test_eq_flat_and_constant(mg):
    procs = mg.ProcessorSet()
    u = np.random.default_rng(7).uniform(-1, 1, size=(1, 2, 4000))
    assert rel(procs.process_node(mg.NodeType.EQ, u, np.zeros(1024)), u) < 1e-5
    assert rel(procs.process_node(mg.NodeType.EQ, u, np.full(1024, -0.4)), u * np.exp(-0.4)) < 1e-5


def test_reverb_kernel_matches_reference(mg, ref):
    for fs in (2000.0, 44100.0):
        procs = mg.ProcessorSet(sample_rate=fs)
        g = mg.Graph()
        g.add_node(mg.NodeType.REVERB)
        gt, ge = g.arrays()
        row = ref.random_legal_params(gt, ge, 11)[8][0]
        l, r = procs.reverb_kernel(row)
        wl, wr = ref.reverb_kernel(row, sample_rate=fs)
        assert rel(l, wl) < TOL and rel(r, wr) < TOL


def test_delay_positions_and_kernel(mg, ref):
    procs = mg.ProcessorSet()
    g = mg.Graph()
    g.add_node(mg.NodeType.DELAY)
    gt, ge = g.arrays()
    for seed in range(5):
        row = ref.random_legal_params(gt, ge, seed)[9][0]
        for c in (0, 1):
            k, pos = ref.delay_kernel(row, c)
            assert procs.delay_positions(row, c) == pos
            assert rel(procs.delay_kernel(row, c), k) < 1e-5
    # test_processors.cpp:388-414
    row = np.zeros(880)
    for tap in range(40):
        row[tap * 22] = 1.0
        row[tap * 22 + 2: tap * 22 + 22] = -80.0

    def enable(r, tap, d, span):
        a = -2 * np.pi * d / span
        r[tap * 22], r[tap * 22 + 1] = np.cos(a), np.sin(a)
        r[tap * 22 + 2: tap * 22 + 22] = 0.0

    enable(row, 0, 100, procs.delay_span)
    enable(row, 1, 4600, procs.delay_span)
    pos = procs.delay_positions(row, 0)
    assert pos[:3] == [100, 4600, -1]
    imp = np.zeros((1, 2, 6000))
    imp[0, 0, 0] = 1.0
    y = procs.process_node(mg.NodeType.DELAY, imp, row)
    assert abs(y[0, 0, 100] - 1.0) < 1e-5 and abs(y[0, 0, 4600] - 1.0) < 1e-5 and abs(y[0, 0, 2000]) < 1e-6


def test_dynamics_long_envelope_correction(mg, ref):
    # alpha -> 1 with envelope_taps < L exercises the a^Ne * e[n-Ne] term of the scan.
    rng = np.random.default_rng(9)
    x = rng.uniform(-1, 1, size=(2, 1, 2, 20000)) * np.linspace(0.01, 1, 20000)
    params = np.array([[0.99995, -2.0, 0.5, 4.0], [0.9999, -1.0, 0.3, 6.0]])
    for t in (5, 6):
        procs = mg.ProcessorSet(sample_rate=44100.0, envelope_taps=4096)
        got = procs.process(t, x, 2, 1, 20000, params, 0)
        want = ref.process(t, x, 2, 1, 20000, params, 0, envelope_taps=4096)
        assert rel(got, want) < TOL


def test_quiet_signal_passes_compressor(mg):
    procs = mg.ProcessorSet()
    u = np.random.default_rng(19).uniform(-1, 1, size=(1, 2, 1000)) * 1e-6
    y = procs.process_node(mg.NodeType.COMPRESSOR, u, [0.99, -1.0, 0.5, 8.0])
    assert np.array_equal(y, u.astype(np.float32).astype(np.float64))


def test_parameter_validation_throws(mg):
    procs = mg.ProcessorSet()
    u = np.zeros((1, 2, 16))
    for bad in ([1.5, -1, 0.5, 4], [0.9, -1, -0.5, 4], [0.9, -1, 0.5, 0.5], [0.9, np.nan, 0.5, 4]):
        with pytest.raises(ValueError):
            procs.process_node(mg.NodeType.COMPRESSOR, u, bad)


# ---- whole renders ---------------------------------------------------------------------------

def test_random_dags_match_reference_and_oracle(mg, ref, procs_small):
    # test_render.cpp:90-106: batched vs per-node reference, fs = 2000, L = 2048.
    for seed in range(13, 21):
        t, e = ref.random_dag(seed, 5, 25)
        params = ref.random_legal_params(t, e, seed)
        src = np.random.default_rng(seed).uniform(-1, 1, size=(int(np.sum(t == 0)), 1, 2, 2048))
        got, want = render_both(mg, ref, t, e, params, src, 2000.0, procs=procs_small)
        assert rel(got, want) < TOL
        slow = ref.render_reference(t, e, params, src, sample_rate=2000.0)
        assert rel(got, slow) < TOL


@pytest.mark.parametrize("strategy", [0, 1, 2, 3])
def test_strategies_render_same_audio(mg, ref, procs_small, strategy):
    for seed in range(40, 44):
        t, e = ref.random_dag(seed, 8, 25)
        params = ref.random_legal_params(t, e, seed)
        src = np.random.default_rng(seed).uniform(-1, 1, size=(int(np.sum(t == 0)), 1, 2, 1024))
        got, want = render_both(mg, ref, t, e, params, src, 2000.0, strategy, procs=procs_small)
        assert rel(got, want) < TOL


def test_config2_full_size_matches_reference(mg, ref):
    # BASELINE config 2: console(16, p=.3, seed=16), stereo 2^17 @ 44.1 kHz, sources as bench.cpp:33-40.
    t, e = ref.console(16, 0.3, 16)
    L = 1 << 17
    params = ref.random_legal_params(t, e, 2024)
    src = np.stack([ref.uniform_noise(2 * L, 1000 + k).reshape(1, 2, L) for k in range(16)])
    got, want = render_both(mg, ref, t, e, params, src, 44100.0)
    assert got.shape == want.shape == (1, 1, 2, L)
    assert rel(got, want) < TOL


def test_config1_chain_matches_reference(mg, ref):
    # BASELINE config 1: in -> (g -> e) x 4 -> out, stereo 2^16.
    g = mg.Graph()
    g.add_serial_chain([0] + [3, 4] * 4 + [1])
    t, e = g.arrays()
    L = 1 << 16
    params = ref.random_legal_params(t, e, 1)
    src = ref.uniform_noise(2 * L, 1000).reshape(1, 1, 2, L)
    got, want = render_both(mg, ref, t, e, params, src, 44100.0)
    assert rel(got, want) < TOL


def test_one_by_one_quirk_renders_like_reference(mg, ref):
    g = mg.Graph()
    for ty in (0, 3, 2, 4, 4, 1):
        g.add_node(ty)
    for s, d in ((0, 1), (1, 2), (1, 2), (0, 3), (3, 4), (4, 2), (2, 5)):
        g.connect(s, d)
    t, e = g.arrays()
    params = ref.random_legal_params(t, e, 5)
    src = np.random.default_rng(5).uniform(-1, 1, size=(1, 1, 2, 3000))
    got, want = render_both(mg, ref, t, e, params, src, 44100.0, strategy=0)
    assert rel(got, want) < TOL


def test_known_answer_renders(mg):
    procs = mg.ProcessorSet()
    rng = np.random.default_rng(3)
    # zero-gain chain is the identity (test_render.cpp:22-32)
    g = mg.Graph()
    g.add_serial_chain([0, 3, 1])
    rd = mg.compute_render_data(mg.to_flat(g))
    s = rng.uniform(-1, 1, size=(1, 1, 2, 1024))
    assert np.array_equal(mg.render(rd, procs, None, s), s.astype(np.float32).astype(np.float64))
    # mix sums, parallel edges double, unconnected nodes are silent (:34-88)
    g = mg.Graph()
    a, b, m, o = g.add_node(0), g.add_node(0), g.add_node(2), g.add_node(1)
    g.connect(a, m)
    g.connect(b, m)
    g.connect(m, o)
    rd = mg.compute_render_data(mg.to_flat(g))
    s = rng.uniform(-1, 1, size=(2, 1, 2, 513)).astype(np.float32).astype(np.float64)
    assert np.array_equal(mg.render(rd, procs, None, s)[0], (s[0] + s[1]).astype(np.float32))
    g = mg.Graph()
    i, m, o = g.add_node(0), g.add_node(2), g.add_node(1)
    g.connect(i, m)
    g.connect(i, m)
    g.connect(m, o)
    rd = mg.compute_render_data(mg.to_flat(g))
    s = rng.uniform(-1, 1, size=(1, 1, 2, 256)).astype(np.float32).astype(np.float64)
    assert np.array_equal(mg.render(rd, procs, None, s)[0], 2 * s[0])
    g = mg.Graph()
    i, o1, eq, o2 = g.add_node(0), g.add_node(1), g.add_node(4), g.add_node(1)
    g.connect(i, o1)
    g.connect(eq, o2)
    rd = mg.compute_render_data(mg.to_flat(g))
    out = mg.render(rd, procs, None, s)
    assert np.array_equal(out[0], s[0]) and not np.any(out[1])


def test_intermediates_in_original_order(mg):
    g = mg.Graph()
    g.add_serial_chain([0, 3, 1])
    fg = mg.to_flat(g)
    fg.params[mg.NodeType.GAIN][0] = np.log(3.0)
    rd = mg.compute_render_data(fg)
    procs = mg.ProcessorSet()
    s = np.random.default_rng(31).uniform(-1, 1, size=(1, 1, 2, 128))
    out, inter = mg.render(rd, procs, None, s, keep_intermediates=True)
    assert inter.shape[0] == 3
    assert rel(inter[0], s[0]) < 1e-7 and np.array_equal(inter[2], out[0])
    assert rel(inter[1], 3 * s[0]) < 1e-6


def test_render_rejects_malformed_inputs(mg):
    g = mg.Graph()
    g.add_serial_chain([0, 3, 1])
    rd = mg.compute_render_data(mg.to_flat(g))
    procs = mg.ProcessorSet()
    with pytest.raises(ValueError):
        mg.render(rd, procs, None, np.zeros((2, 1, 2, 64)))
    bad = {k: v.copy() for k, v in rd.flat.params.items()}
    bad[mg.NodeType.GAIN][0, 0] = np.nan
    with pytest.raises(ValueError):
        mg.render(rd, procs, bad, np.zeros((1, 1, 2, 64)))


def test_union_renders_like_parts(mg, ref, procs_small):
    # test_render.cpp:132-160
    t1, e1 = ref.random_dag(19, 5, 15)
    t2, e2 = ref.random_dag(20, 5, 15)
    g = mg.disjoint_union([mg.Graph.from_arrays(t1, e1), mg.Graph.from_arrays(t2, e2)])
    tu, eu = g.arrays()
    p1, p2 = ref.random_legal_params(t1, e1, 1), ref.random_legal_params(t2, e2, 2)
    pu = mg.concat_params([p1, p2])
    rng = np.random.default_rng(19)
    s1 = rng.uniform(-1, 1, size=(int(np.sum(t1 == 0)), 1, 2, 1024))
    s2 = rng.uniform(-1, 1, size=(int(np.sum(t2 == 0)), 1, 2, 1024))
    r1, _ = render_both(mg, ref, t1, e1, p1, s1, 2000.0, procs=procs_small)
    r2, _ = render_both(mg, ref, t2, e2, p2, s2, 2000.0, procs=procs_small)
    ru, _ = render_both(mg, ref, tu, eu, pu, np.concatenate([s1, s2]), 2000.0, procs=procs_small)
    assert rel(ru[: len(r1)], r1) < 1e-6 and rel(ru[len(r1):], r2) < 1e-6


def test_batch_equals_singles(mg, ref, procs_small):
    # test_render.cpp:162-192 (source-level batching)
    t, e = ref.random_dag(23, 6, 20)
    params = ref.random_legal_params(t, e, 23)
    fg = make(mg, t, e)
    rd = mg.compute_render_data(fg)
    P = rd.reorder_params(params)
    src = np.random.default_rng(23).uniform(-1, 1, size=(int(np.sum(t == 0)), 3, 2, 800))
    big = mg.render(rd, procs_small, P, src)
    for b in range(3):
        one = mg.render(rd, procs_small, P, src[:, b:b + 1])
        assert np.max(np.abs(big[:, b] - one[:, 0])) < 1e-6


def test_lti_graph_is_linear(mg, ref, procs_small):
    g = mg.Graph()
    i = g.add_node(0)
    a, b = g.add_serial_chain([4, 7, 3, 9])
    o = g.add_node(1)
    g.connect(i, a)
    g.connect(b, o)
    g.connect(i, o)
    t, e = g.arrays()
    params = ref.random_legal_params(t, e, 29)
    rd = mg.compute_render_data(make(mg, t, e))
    P = rd.reorder_params(params)
    rng = np.random.default_rng(29)
    s1, s2 = rng.uniform(-1, 1, size=(2, 1, 1, 2, 1024))
    y = mg.render(rd, procs_small, P, 0.8 * s1 - 0.6 * s2)
    y1, y2 = mg.render(rd, procs_small, P, s1), mg.render(rd, procs_small, P, s2)
    assert rel(y, 0.8 * y1 - 0.6 * y2) < TOL


def test_device_path_equals_host_path(mg, ref):
    import torch
    t, e = ref.console(4, 0.0, 3)
    L = 20000
    params = ref.random_legal_params(t, e, 4)
    rd = mg.compute_render_data(make(mg, t, e))
    procs = mg.ProcessorSet()
    P = rd.reorder_params(params)
    src = np.random.default_rng(4).uniform(-1, 1, size=(rd.num_inputs, 1, 2, L))
    host = mg.render(rd, procs, P, src)
    dr = mg.DeviceRenderer(rd, procs, 1, L, P)
    dr.sources.copy_(torch.as_tensor(src, dtype=torch.float32))
    out = dr.render().cpu().numpy()
    torch.cuda.synchronize()
    assert np.array_equal(out, host.astype(np.float32))
    want = ref.Plan(t, e, 1).render(params, src)
    assert rel(out, want) < TOL


def test_renders_are_bit_reproducible(mg, ref):
    # The envelope scan's cross-tile carry is a fixed-order sum: repeated renders are identical.
    t, e = ref.console(8, 0.3, 5)
    params = ref.random_legal_params(t, e, 6)
    rd = mg.compute_render_data(make(mg, t, e))
    procs = mg.ProcessorSet()
    P = rd.reorder_params(params)
    src = np.random.default_rng(6).uniform(-1, 1, size=(rd.num_inputs, 2, 2, 70000))
    first = mg.render(rd, procs, P, src)
    for _ in range(3):
        assert np.array_equal(mg.render(rd, procs, P, src), first)


@pytest.mark.parametrize("dtype,host_threads", [(np.float32, -1), (np.float64, -1), (np.float64, 0)])
def test_render_pipeline_matches_render(mg, ref, dtype, host_threads):
    # Streaming host API: back-to-back submits with different sources and parameters; with
    # depth 2 the third and fourth reuse slots whose previous outputs may still be in flight
    # (host_threads=0: double audio converted on the device, outputs staged beside the next
    # sources in the same device buffer).
    t, e = ref.console(3, 0.0, 9)
    L = 30000
    rd = mg.compute_render_data(make(mg, t, e))
    procs = mg.ProcessorSet()
    pipe = mg.RenderPipeline(rd, procs, 1, L, dtype=dtype, depth=2, host_threads=host_threads)
    cases = []
    for i in range(5):
        P = rd.reorder_params(ref.random_legal_params(t, e, 100 + i))
        src = pipe.pinned((rd.num_inputs, 1, 2, L))
        src[...] = np.random.default_rng(i).uniform(-1, 1, size=src.shape)
        out = pipe.pinned((1, 1, 2, L))
        pipe.submit(P, src, out)
        cases.append((P, np.array(src, dtype=np.float64), out))
    pipe.sync()
    for P, src, out in cases:
        want = mg.render(rd, procs, P, src.astype(np.float32).astype(np.float64))
        assert np.array_equal(out.astype(np.float64), want.astype(np.float32).astype(np.float64)) if dtype == np.float32 \
            else np.array_equal(out, want)


def _random_union(mg, sharding, seed, graphs):
    rng = np.random.default_rng(seed)
    members = [wl.generate_console_arrays(int(rng.integers(2, 9)), 0.3, 50 * seed + i) for i in range(graphs)]
    return sharding.union_arrays(members)


@pytest.mark.parametrize("on_device", [True, False])
def test_batch_renderer_redrawn_topologies(mg, ref, on_device):
    # Config-3 style: a different union every submit, original-order parameters reordered on
    # the device, sources cycled from a bank; every render equals the blocking render().
    import torch
    from paper_2408_03204_b200 import sharding
    L = 12000
    procs = mg.ProcessorSet()
    bank = np.random.default_rng(1).uniform(-1, 1, size=(5, 1, 2, L)).astype(np.float32)
    batches = []
    for i in range(4):
        t, e = _random_union(mg, sharding, i, 3 + i)
        batches.append((t, e, mg.compute_render_data_arrays(t, e), wl.random_legal_params(t, 70 + i)))
    cap = np.zeros(4, dtype=np.uint64)
    for _, _, rd, _ in batches:
        cap = np.maximum(cap, mg.BatchRenderer.capacity_of(rd, procs, 1, L))
    br = mg.BatchRenderer(procs, 1, L, cap, depth=2)
    src = torch.as_tensor(bank).cuda() if on_device else bank
    outs = []
    for t, e, rd, params in batches:
        out = np.zeros((rd.buffer_rows - rd.output_begin, 1, 2, L), dtype=np.float32)
        br.submit(rd, params, src, out)
        outs.append(out)
    br.sync()
    for (t, e, rd, params), out in zip(batches, outs):
        k = rd.num_inputs
        s = bank[np.arange(k) % len(bank)].astype(np.float64)
        want = mg.render(rd, procs, rd.reorder_params(params), s)
        assert np.array_equal(out.astype(np.float64), want)
    t, e, rd, params = batches[-1]
    assert rel(outs[-1], ref.Plan(t, e, 1).render(params, bank[np.arange(rd.num_inputs) % 5].astype(np.float64))) < TOL
    dev_out = br.last_outputs().cpu().numpy()
    assert np.array_equal(dev_out, outs[-1])


def test_batch_renderer_rejects_bad_params(mg):
    from paper_2408_03204_b200 import sharding
    L = 4096
    procs = mg.ProcessorSet()
    t, e = _random_union(mg, sharding, 9, 2)
    rd = mg.compute_render_data_arrays(t, e)
    br = mg.BatchRenderer(procs, 1, L, mg.BatchRenderer.capacity_of(rd, procs, 1, L))
    src = np.zeros((1, 1, 2, L), dtype=np.float32)
    params = wl.random_legal_params(t, 3)
    bad = {k: v.copy() for k, v in params.items()}
    bad[mg.NodeType.COMPRESSOR][0, 0] = 1.5
    with pytest.raises(ValueError, match="alpha"):
        br.submit(rd, bad, src)
    short = {k: v for k, v in params.items() if k != mg.NodeType.EQ}
    with pytest.raises(ValueError, match="missing or misshaped"):
        br.submit(rd, short, src)
    br.submit(rd, params, src)
    br.sync()


def _track_params(mg, t, params, tracks, k):
    """Parameter rows of track k of generate_large_console(tracks), as a 1-track table set
    (rows of each type are numbered in node insertion order; tracks come first)."""
    per = {}
    for ty in set(int(x) for x in t[:15]):
        if mg.param_width(ty):
            per[ty] = int(np.sum(t[:15] == ty))
    small = {}
    for ty, n in per.items():
        tab = params[mg.NodeType(ty)]
        small[mg.NodeType(ty)] = tab[k * n:(k + 1) * n]
    # bus rows (one eq, comp, imager, gain) follow all track rows of their type
    for ty in (mg.NodeType.EQ, mg.NodeType.COMPRESSOR, mg.NodeType.IMAGER, mg.NodeType.GAIN):
        n = per[int(ty)]
        small[ty] = np.concatenate([small[ty], params[ty][tracks * n:tracks * n + 1]])
    return small


def test_config4_large_graph_full_size(mg, ref):
    # BASELINE config 4: 64 tracks, 966 nodes, 10 s stereo (L = 441000, 2^20-point reverb
    # convolutions). The full graph is checked track by track: each track's strip and send
    # outputs (intermediates) equal a 1-track graph rendered with that track's parameters,
    # and the 1-track graph matches the reference renderer at full length.
    L, tracks = 441000, 64
    t, e = wl.generate_large_console_arrays(tracks)
    assert len(t) == 966 and len(e) == 1093
    params = wl.random_legal_params(t, 44)
    k_src = 3
    src = np.stack([mg.uniform_noise(2 * L, 1000 + (k % k_src)).reshape(1, 2, L) for k in range(tracks)])
    import torch
    procs = mg.ProcessorSet()
    rd = mg.compute_render_data_arrays(t, e)
    dr = mg.DeviceRenderer(rd, procs, 1, L, rd.reorder_params(params))
    dr.sources.copy_(torch.as_tensor(src, dtype=torch.float32))
    out = dr.render().cpu().numpy()
    assert np.isfinite(out).all() and np.abs(out).max() > 0
    sigma = np.asarray(rd.sigma)
    t1, e1 = wl.generate_large_console_arrays(1)
    rd1 = mg.compute_render_data_arrays(t1, e1)
    for k in (0, 37, 63):
        p1 = _track_params(mg, t, params, tracks, k)
        y1, i1 = mg.render(rd1, procs, rd1.reorder_params(p1), src[k:k + 1], keep_intermediates=True)
        rows = torch.as_tensor(sigma[15 * k:15 * k + 15], device=dr.arena.device)
        big = dr.arena.index_select(0, rows).cpu().numpy()
        assert rel(big, i1[:15]) < 1e-5, k
        if k == 37:
            want = ref.Plan(t1, e1, 1).render(p1, src[k:k + 1])
            assert rel(y1, want) < TOL


@pytest.mark.parametrize("L", [8192, 7000])
def test_fused_kernel_rows_match_separate_pass(mg, ref, L):
    # Large conv steps transform the kernel rows inside the signal's row pass; forced both
    # ways on a console the renders agree, and so do the backward passes.
    import torch
    t, e = ref.console(6, 0.0, 4)
    params = ref.random_legal_params(t, e, 5)
    rd = mg.compute_render_data(make(mg, t, e))
    procs = mg.ProcessorSet()
    P = rd.reorder_params(params)
    src = np.random.default_rng(L).uniform(-1, 1, size=(rd.num_inputs, 1, 2, L))
    res = []
    try:
        for mode in (0, 1):
            mg.set_conv_fuse(mode)
            dr = mg.DeviceRenderer(rd, procs, 1, L, P, backward=True)
            dr.sources.copy_(torch.as_tensor(src, dtype=torch.float32))
            out = dr.render().clone()
            w = torch.ones_like(out)
            g, gs = dr.backward(w)
            torch.cuda.synchronize()
            res.append((out.cpu().numpy(), {k: v.cpu().numpy() for k, v in g.items()}, gs.cpu().numpy()))
    finally:
        mg.set_conv_fuse(-1)
    (o0, g0, s0), (o1, g1, s1) = res
    assert rel(o1, o0) < 1e-5 and rel(s1, s0) < 1e-5
    for k in g0:
        assert rel(g1[k], g0[k]) < 1e-4, k  # fp32 noise of small delay gradients (see test_backward_gpu)
    assert rel(o0, ref.Plan(t, e, 1).render(params, src)) < TOL


@pytest.mark.parametrize("tracks,L,batch", [(8, 70000, 2), (8, 70001, 1), (3, 4093, 2)])
def test_pointwise_epilogue_fusion_is_bit_exact(mg, ref, tracks, L, batch):
    # Pointwise follower steps (the per-track noisegate -> imager -> gain chain, the bus tail
    # compressor -> imager -> gain -> out) ride in the previous step's epilogue in render();
    # render_profiled() launches every step on its own. Every arena row must be identical.
    import torch
    from paper_2408_03204_b200.device import DeviceRenderer
    t, e = ref.console(tracks, 0.3, 7)
    params = ref.random_legal_params(t, e, 8)
    rd = mg.compute_render_data(make(mg, t, e))
    procs = mg.ProcessorSet()
    P = rd.reorder_params(params)
    src = np.random.default_rng(3).uniform(-1, 1, size=(rd.num_inputs, batch, 2, L))
    dr = DeviceRenderer(rd, procs, batch, L, P)
    dr.sources.copy_(torch.as_tensor(src, dtype=torch.float32))
    dr.render()
    fused = dr.arena.clone()
    dr.arena[rd.num_inputs:].fill_(float("nan"))
    dr.render_profiled(sync=True)
    torch.cuda.synchronize()
    assert torch.equal(fused.view(torch.int32), dr.arena.view(torch.int32))
    want = ref.Plan(t, e, 1).render(params, src)
    assert rel(fused[rd.output_begin:].cpu().numpy(), want) < TOL


def test_fp64_transforms_config2(mg, ref):
    # The fp64-arithmetic mode of every FFT-based step (EQ, reverb, delay) on config 2 at full
    # size; the EQ steps' own error drops ~2x (arena and the other processors stay fp32).
    t, e, params = wl.config2()
    L = wl.L2
    src = wl.sources(int(np.sum(t == 0)), L)
    rd = mg.compute_render_data_arrays(t, e)
    procs = mg.ProcessorSet()
    want = ref.Plan(t, e, 1).render(params, src)
    mg.set_fft_precision(64)
    try:
        assert mg.fft_precision() == 64
        y = mg.render(rd, procs, rd.reorder_params(params), src)
    finally:
        mg.set_fft_precision(32)
    assert rel(y, want) < TOL


def test_step_owners_and_serialized_render(mg, ref):
    # step_owners: which launch computes each step (measurement attribution). A serialised
    # render (render_profiled(hoist=False) without step times: prologues inline, no side
    # streams) runs the same kernels, so its arena equals the overlapped render's bit for bit.
    import torch
    from paper_2408_03204_b200.device import DeviceRenderer
    t, e = ref.console(6, 0.3, 5)
    params = ref.random_legal_params(t, e, 9)
    rd = mg.compute_render_data(make(mg, t, e))
    L = 20000
    own = rd.step_owners(1, L)
    assert len(own) == rd.num_steps
    for k, o in enumerate(own):
        assert 0 <= o <= k and own[o] == o
        if o != k:  # followers are pointwise types
            assert int(rd.steps[k].type) in (1, 2, 3, 7)
    types = [int(st.type) for st in rd.steps]
    gate = types.index(6)
    assert own[gate + 1] == gate  # the per-track imager rides in the noisegate scan's epilogue
    procs = mg.ProcessorSet()
    src = np.random.default_rng(4).uniform(-1, 1, size=(rd.num_inputs, 1, 2, L))
    dr = DeviceRenderer(rd, procs, 1, L, rd.reorder_params(params))
    dr.sources.copy_(torch.as_tensor(src, dtype=torch.float32))
    dr.render()
    a = dr.arena.clone()
    dr.arena[rd.num_inputs:].fill_(float("nan"))
    dr.render_profiled(hoist=False)
    torch.cuda.synchronize()
    assert torch.equal(a.view(torch.int32), dr.arena.view(torch.int32))


@pytest.mark.parametrize("taps,L", [(None, 70000), (4096, 20000), (4097, 20000), (4096, 12), (4096, 20004)])
def test_streaming_scan_matches_reference(mg, ref, taps, L):
    # The compressor / noisegate scan forced onto the streaming kernel (one CTA per sequence,
    # bulk-copy ring, running carry) and onto the chained look-back scan: both match the
    # reference, and each other to fp64 rounding of the envelope. envelope_taps < L exercises
    # the a^Ne correction (4097: its unaligned re-gather); L = 12: one partial tile.
    rng = np.random.default_rng(L + (taps or 0))
    slots, batch = 5, 2
    x = rng.uniform(-1, 1, size=(slots, batch, 2, L)) * np.linspace(0.01, 1, L)
    cfg = {} if taps is None else {"envelope_taps": taps}
    for t in (5, 6):
        g = mg.Graph()
        for _ in range(slots):
            g.add_node(t)
        gt, ge = g.arrays()
        params = ref.random_legal_params(gt, ge, 77 + t)[t]
        params[:, 0] = np.linspace(0.9, 0.9999, slots)
        procs = mg.ProcessorSet(sample_rate=44100.0, **cfg)
        want = ref.process(t, x, slots, batch, L, params, 0, **cfg)
        got = {}
        for mode in (1, 0):
            mg.set_dyn_stream(mode)
            try:
                got[mode] = procs.process(t, x, slots, batch, L, params, 0)
            finally:
                mg.set_dyn_stream(-1)
            assert rel(got[mode], want) < TOL, (t, mode)
        assert rel(got[1], got[0]) < 1e-5


@pytest.mark.parametrize("prune,L,batch", [(0.0, 20000, 1), (0.4, 9000, 2)])
def test_shared_signal_spectra_bit_exact(mg, ref, prune, L, batch):
    # A console track's gain feeds its delay and its reverb: with the kernel rows fused into the
    # row pass (forced here; automatic for config-5-sized steps), the second conv step reuses
    # the first one's signal spectra for those tracks (launch_conv_shared). render_profiled()
    # runs every step on its own (no sharing): the arenas must be bit-identical.
    import torch
    from paper_2408_03204_b200.device import DeviceRenderer
    t, e = ref.console(6, prune, 11)
    params = ref.random_legal_params(t, e, 12)
    rd = mg.compute_render_data(make(mg, t, e))
    types = [int(st.type) for st in rd.steps]
    k = next(i for i in range(1, len(types)) if {types[i - 1], types[i]} == {8, 9})
    assert k > 0
    procs = mg.ProcessorSet()
    src = np.random.default_rng(5).uniform(-1, 1, size=(rd.num_inputs, batch, 2, L))
    assert rd.shared_pairs(procs, batch, L)[k] == 0  # small steps: separate (side-by-side) passes
    mg.set_conv_fuse(1)
    try:
        pairs = rd.shared_pairs(procs, batch, L)
        assert pairs[k] > 0 and pairs.sum() == pairs[k]
        dr = DeviceRenderer(rd, procs, batch, L, rd.reorder_params(params))
        dr.sources.copy_(torch.as_tensor(src, dtype=torch.float32))
        dr.render()
        shared = dr.arena.clone()
        dr.arena[rd.num_inputs:].fill_(float("nan"))
        dr.render_profiled(sync=True)
        torch.cuda.synchronize()
        assert torch.equal(shared.view(torch.int32), dr.arena.view(torch.int32))
        g = dr.capture()
        dr.arena[rd.num_inputs:].fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(shared.view(torch.int32), dr.arena.view(torch.int32))
    finally:
        mg.set_conv_fuse(-1)
    want = ref.Plan(t, e, 1).render(params, src)
    assert rel(shared[rd.output_begin:].cpu().numpy(), want) < TOL


@pytest.mark.parametrize("taps,L", [(None, 20000), (4096, 20000), (4097, 12000), (600, 9000), (4096, 9004)])
def test_fused_compressor_gate_scan(mg, ref, taps, L):
    # A console track's compressor -> noisegate (-> imager -> gain) as ONE streaming kernel
    # (forced onto the streaming path; automatic for config-5-sized steps): matches the
    # reference, the two-launch streaming path and the chained scans; envelope_taps < L
    # exercises both stages' a^Ne re-gathers (600: within the same tile).
    import torch
    from paper_2408_03204_b200.device import DeviceRenderer
    t, e = ref.console(5, 0.3, 21)
    params = ref.random_legal_params(t, e, 22)
    for ty in (5, 6):
        params[ty][:, 0] = np.linspace(0.99, 0.9999, len(params[ty]))
    rd = mg.compute_render_data(make(mg, t, e))
    cfg = {} if taps is None else {"envelope_taps": taps}
    procs = mg.ProcessorSet(**cfg)
    src = np.random.default_rng(23).uniform(-1, 1, size=(rd.num_inputs, 1, 2, L)) * np.linspace(0.01, 1, L)
    dr = DeviceRenderer(rd, procs, 1, L, rd.reorder_params(params))
    dr.sources.copy_(torch.as_tensor(src, dtype=torch.float32))
    arenas = {}
    try:
        for mode in ((1, 1), (1, 0), (0, 0)):
            mg.set_dyn_stream(mode[0])
            mg.set_dyn_pair(mode[1])
            dr.arena[rd.num_inputs:].fill_(float("nan"))
            dr.render()
            torch.cuda.synchronize()
            arenas[mode] = dr.arena.clone()
    finally:
        mg.set_dyn_stream(-1)
        mg.set_dyn_pair(-1)
    assert torch.equal(arenas[(1, 1)].view(torch.int32), arenas[(1, 0)].view(torch.int32))
    want = ref.Plan(t, e, 1).render(params, src, **cfg)
    for mode, a in arenas.items():
        assert rel(a[rd.output_begin:].cpu().numpy(), want) < TOL, mode


def test_serialized_render_equals_fused_render_all_paths(mg, ref):
    # bench.py's per-kernel roofline trace renders with hoist=False (everything on one stream):
    # with the shared delay/reverb spectra, the fused compressor -> noisegate scan and the
    # epilogue followers all active (forced here), its arena must equal the overlapped render's.
    import torch
    from paper_2408_03204_b200.device import DeviceRenderer
    t, e = ref.console(7, 0.2, 31)
    params = ref.random_legal_params(t, e, 32)
    rd = mg.compute_render_data(make(mg, t, e))
    L = 24000
    procs = mg.ProcessorSet()
    src = np.random.default_rng(33).uniform(-1, 1, size=(rd.num_inputs, 1, 2, L))
    mg.set_conv_fuse(1)
    mg.set_dyn_stream(1)
    try:
        assert rd.shared_pairs(procs, 1, L).sum() > 0
        own = rd.step_owners(1, L)
        types = [int(st.type) for st in rd.steps]
        assert own[types.index(6)] == types.index(5)  # the noisegate runs in the compressor's launch
        dr = DeviceRenderer(rd, procs, 1, L, rd.reorder_params(params))
        dr.sources.copy_(torch.as_tensor(src, dtype=torch.float32))
        g = dr.capture()
        g.replay()
        torch.cuda.synchronize()
        a = dr.arena.clone()
        dr.arena[rd.num_inputs:].fill_(float("nan"))
        dr.render_profiled(hoist=False)
        torch.cuda.synchronize()
        assert torch.equal(a.view(torch.int32), dr.arena.view(torch.int32))
    finally:
        mg.set_conv_fuse(-1)
        mg.set_dyn_stream(-1)
    want = ref.Plan(t, e, 1).render(params, src)
    assert rel(a[rd.output_begin:].cpu().numpy(), want) < TOL
