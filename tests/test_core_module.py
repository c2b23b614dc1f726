"""mixgraph._core, the pybind11 module the reference declares (`proj/CMakeLists.txt:47-74`;
its tests/CMakeLists.txt:26-34 runs a python_smoke over it), built by build() over the
product's C++ API. Host-side parity with the reference on CPU; the render on the GPU."""
import numpy as np
import pytest

from conftest import cuda_ok

core = pytest.importorskip("mixgraph")


def console_graph(ref, tracks, prune, seed):
    t, e = ref.console(tracks, prune, seed)
    g = core.Graph()
    for x in t:
        g.add_node(core.NodeType(int(x)))
    for s, d, o, i in e:
        g.connect(int(s), int(d), int(o), int(i))
    return g, t, e


def test_core_schedule_matches_reference(ref):
    g, t, e = console_graph(ref, 16, 0.3, 16)
    fg = core.to_flat(g)
    assert fg.num_nodes() == 121 and fg.num_inputs == 16 and fg.num_outputs == 1
    for strategy, codes in ((core.Strategy.Greedy, "iecnsgrdmecsgo"), (core.Strategy.Beam, "iecnsgdrmecsgo")):
        rd = core.compute_render_data(fg, core.ScheduleOptions(strategy=strategy))
        want = ref.Plan(t, e, int(strategy))
        assert rd.schedule.type_codes() == codes == want.type_codes
        assert list(rd.sigma) == want.sigma
        assert rd.buffer_rows == want.buffer_rows and rd.output_begin == want.output_begin
        for st, ws in zip(rd.steps, want.steps):
            assert (int(st.type), list(st.gather), list(st.aggregate), st.store_begin, st.store_end) == \
                (ws["type"], ws["gather"], ws["aggregate"], ws["store_begin"], ws["store_end"])


def test_core_errors_are_value_errors():
    g = core.Graph()
    a, b = g.add("gain"), g.add("eq")
    g.connect(a, b)
    g.connect(b, a)
    with pytest.raises(ValueError, match="cycle"):
        g.validate()
    with pytest.raises(ValueError, match="unknown node type"):
        core.Graph().add("flanger")


def test_core_reorder_params_round_trip(ref):
    g, t, e = console_graph(ref, 4, 0.0, 1)
    rd = core.compute_render_data(core.to_flat(g))
    params = {core.NodeType(int(k)): v for k, v in ref.random_legal_params(t, e, 3).items()}
    re = rd.reorder_params(params)
    for ty, rows in rd.param_source_rows.items():
        assert np.array_equal(re[ty], params[ty][np.asarray(rows)])


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")
def test_core_render_matches_abi_and_reference(mg, ref):
    g, t, e = console_graph(ref, 4, 0.3, 7)
    rd = core.compute_render_data(core.to_flat(g))
    params = ref.random_legal_params(t, e, 11)
    L = 20000
    src = np.random.default_rng(2).uniform(-1, 1, size=(4, 1, 2, L))
    procs = core.ProcessorSet(core.ProcessorConfig(sample_rate=44100.0))
    out, inter = core.render_grafx(src, procs, {core.NodeType(int(k)): v for k, v in params.items()}, rd,
                                   keep_intermediates=True)
    assert out.shape == (1, 1, 2, L) and inter.shape == (len(t), 1, 2, L)
    rd_abi = mg.compute_render_data_arrays(t, e)
    y_abi = mg.render(rd_abi, mg.ProcessorSet(), rd_abi.reorder_params(params), src)
    assert np.array_equal(out, y_abi)
    assert ref.rel_linf(out, ref.Plan(t, e, 1).render(params, src)) < 1e-4
