"""Render-order computation: bit-exact parity of the C++ plan builder with the reference.

Compares every field of RenderData (schedule type string + subsets, sigma, reordered
graph, every StepIndex, param_source_rows) between the product (libmgb200.so through the
C ABI) and the compiled reference (oracle/_ref), for all four strategies, on the graph
families the reference's own tests use (`proj/tests/test_schedule.cpp`): random DAGs from
`testutil::random_dag`, consoles, disjoint unions and the Fig. 1 snippet.
"""
import numpy as np
import pytest

STRATS = [0, 1, 2, 3]


def plan_pair(mg, ref, t, e, strategy, beam=32, cap=256):
    fg = mg.to_flat(mg.Graph.from_arrays(t, e))
    rd = mg.compute_render_data(fg, strategy, beam, cap)
    rp = ref.Plan(t, e, strategy, beam, cap)
    return rd, rp


def assert_same(rd, rp):
    assert rd.schedule.type_codes() == rp.type_codes
    assert rd.schedule.subsets == rp.subsets
    assert rd.sigma == rp.sigma
    assert [int(x) for x in rd.flat.node_types] == rp.flat_types
    assert [tuple(x) for x in rd.flat.edges] == rp.flat_edges
    assert (rd.buffer_rows, rd.num_inputs, rd.output_begin) == (rp.buffer_rows, rp.num_inputs, rp.output_begin)
    assert len(rd.steps) == len(rp.steps)
    for a, b in zip(rd.steps, rp.steps):
        assert int(a.type) == b["type"]
        assert (a.param_begin, a.param_end, a.store_begin, a.store_end) == (
            b["param_begin"], b["param_end"], b["store_begin"], b["store_end"])
        assert a.gather == b["gather"]
        assert a.aggregate == b["aggregate"]
    assert {int(k): v for k, v in rd.param_source_rows.items()} == rp.param_source_rows


@pytest.mark.parametrize("strategy", STRATS)
def test_random_dags_match_reference(mg, ref, strategy):
    for seed in range(120):
        t, e = ref.random_dag(seed, 5, 40, heavy=seed % 2 == 0)
        rd, rp = plan_pair(mg, ref, t, e, strategy)
        assert_same(rd, rp)


@pytest.mark.parametrize("strategy", STRATS)
def test_consoles_match_reference(mg, ref, strategy):
    for k in (1, 2, 3, 4, 8, 16, 31):
        for prune, seed in ((0.0, 0), (0.3, 16), (0.5, 7)):
            t, e = ref.console(k, prune, seed)
            rd, rp = plan_pair(mg, ref, t, e, strategy)
            assert_same(rd, rp)


def test_config2_console_step_table(mg, ref):
    # BASELINE config 2: generate_console(16, {p=0.3, seed=16}) -> 121 nodes, 139 edges, 13 steps.
    t, e = ref.console(16, 0.3, 16)
    assert (len(t), len(e)) == (121, 139)
    rd, rp = plan_pair(mg, ref, t, e, 1)
    assert_same(rd, rp)
    assert rd.schedule.type_codes() == "iecnsgrdmecsgo"
    assert [len(s.gather) for s in rd.steps] == [16, 16, 16, 16, 16, 12, 7, 35, 1, 1, 1, 1, 1]


@pytest.mark.parametrize("strategy", [1, 2])
def test_unions_match_reference(mg, ref, strategy):
    rng = np.random.default_rng(5)
    types, edges, off = [], [], 0
    for i in range(24):
        t, e = ref.console(int(rng.integers(4, 33)), 0.3, 1000 + i)
        types.append(t)
        edges.append(e + np.array([off, off, 0, 0], dtype=np.int32))
        off += len(t)
    t = np.concatenate(types)
    e = np.concatenate(edges)
    rd, rp = plan_pair(mg, ref, t, e, strategy)
    assert_same(rd, rp)


def test_fig1_snippet(mg, ref):
    t, e = ref.four_track_snippet()
    assert len(t) == 21
    for s in STRATS:
        rd, rp = plan_pair(mg, ref, t, e, s)
        assert_same(rd, rp)
    rd, _ = plan_pair(mg, ref, t, e, 3)
    assert rd.schedule.num_steps() == 9
    assert rd.schedule.type_codes() == "iecgmregro"


def test_beam_widths_match_reference(mg, ref):
    for seed in range(20):
        t, e = ref.random_dag(1000 + seed, 8, 32)
        for w in (1, 2, 4, 8, 16, 32):
            rd, rp = plan_pair(mg, ref, t, e, 2, beam=w)
            assert_same(rd, rp)


def test_one_by_one_parallel_edge_quirk(mg, ref):
    # Parallel interior edges decrement the one-by-one in-degree once per EDGE
    # (schedule.cpp:186-203), so b (row 2) is emitted before its other predecessor c.
    g = mg.Graph()
    for t in (mg.NodeType.IN, mg.NodeType.GAIN, mg.NodeType.MIX, mg.NodeType.EQ, mg.NodeType.EQ, mg.NodeType.OUT):
        g.add_node(t)
    for s, d in ((0, 1), (1, 2), (1, 2), (0, 3), (3, 4), (4, 2), (2, 5)):
        g.connect(s, d)
    t, e = g.arrays()
    rd, rp = plan_pair(mg, ref, t, e, 0)
    assert_same(rd, rp)
    assert rd.schedule.subsets[1:3] == [[1], [2]]


def test_graph_errors_match_reference(mg, ref):
    cases = []
    # cycle
    cases.append(([4, 4], [[0, 1, 0, 0], [1, 0, 0, 0]]))
    # cycle downstream witness
    cases.append(([0, 4, 4, 3, 1], [[0, 1, 0, 0], [1, 2, 0, 0], [2, 1, 0, 0], [2, 3, 0, 0], [3, 4, 0, 0]]))
    # channel
    cases.append(([4, 4], [[0, 1, 0, 1]]))
    for t, e in cases:
        t = np.asarray(t, dtype=np.int32)
        e = np.asarray(e, dtype=np.int32)
        with pytest.raises(ValueError) as want:
            ref.Plan(t, e, 1)
        with pytest.raises(ValueError) as got:
            mg.compute_render_data(mg.FlatGraph([mg.NodeType(x) for x in t], [tuple(r) for r in e]), 1)
        assert str(got.value) == str(want.value)
    assert "cycle" in str(pytest.raises(ValueError, mg.Graph.from_arrays([4, 4], [[0, 1, 0, 0], [1, 0, 0, 0]]).validate).value)


def test_optimal_cap_mentions_beam(mg, ref):
    g = mg.Graph()
    i = g.add_node(mg.NodeType.IN)
    m = g.add_node(mg.NodeType.MIX)
    g.connect(i, m)
    for _ in range(300):
        g.connect(m, g.add_node(mg.NodeType.GAIN))
    fg = mg.to_flat(g)
    with pytest.raises(ValueError, match="beam") as got:
        mg.compute_render_data(fg, mg.Strategy.OPTIMAL)
    t, e = g.arrays()
    with pytest.raises(ValueError) as want:
        ref.Plan(t, e, 3)
    assert str(got.value) == str(want.value)
    rd = mg.compute_render_data(fg, mg.Strategy.OPTIMAL, optimal_node_cap=512)
    assert rd.schedule.num_steps() == 2


def test_validate_schedule_names_condition(mg):
    # test_schedule.cpp:83-113
    g = mg.Graph()
    g.add_serial_chain([mg.NodeType.IN, mg.NodeType.GAIN, mg.NodeType.OUT])
    fg = mg.to_flat(g)
    s = mg.make_schedule(fg, mg.Strategy.GREEDY)
    mg.validate_schedule(fg, s)
    rev = mg.Schedule(list(s.type_string), [s.subsets[0], s.subsets[2], s.subsets[1]])
    with pytest.raises(ValueError, match="homogeneity"):
        mg.validate_schedule(fg, rev)
    g2 = mg.Graph()
    g2.add_serial_chain([mg.NodeType.IN, mg.NodeType.EQ, mg.NodeType.GAIN, mg.NodeType.OUT])
    fg2 = mg.to_flat(g2)
    N = mg.NodeType
    with pytest.raises(ValueError, match="causality"):
        mg.validate_schedule(fg2, mg.Schedule([N.IN, N.GAIN, N.EQ, N.OUT], [[0], [2], [1], [3]]))
    with pytest.raises(ValueError, match="homogeneity"):
        mg.validate_schedule(fg2, mg.Schedule([N.IN, N.EQ, N.OUT], [[0], [1, 2], [3]]))
    with pytest.raises(ValueError, match="empty"):
        mg.validate_schedule(fg2, mg.Schedule([N.IN, N.EQ, N.GAIN, N.OUT], [[0], [1], [2], []]))


def test_chain_indices_and_parallel_edges(mg):
    # test_schedule.cpp:222-250
    g = mg.Graph()
    g.add_serial_chain([mg.NodeType.IN, mg.NodeType.GAIN, mg.NodeType.OUT])
    rd = mg.compute_render_data(mg.to_flat(g))
    assert [(s.gather, s.aggregate, s.store_begin, s.store_end) for s in rd.steps] == [([0], [0], 1, 2), ([1], [0], 2, 3)]
    assert (rd.steps[0].param_begin, rd.steps[0].param_end, rd.buffer_rows) == (0, 1, 3)
    g = mg.Graph()
    i, m, o = g.add_node(mg.NodeType.IN), g.add_node(mg.NodeType.MIX), g.add_node(mg.NodeType.OUT)
    g.connect(i, m)
    g.connect(i, m)
    g.connect(m, o)
    rd = mg.compute_render_data(mg.to_flat(g))
    assert rd.steps[0].gather == [0, 0] and rd.steps[0].aggregate == [0, 0]


def test_strategy_quality_ordering(mg, ref):
    # test_schedule.cpp:124-138 on the product
    for seed in range(40):
        t, e = ref.random_dag(3000 + seed, 5, 40)
        fg = mg.to_flat(mg.Graph.from_arrays(t, e))
        n = [mg.make_schedule(fg, s).num_steps() for s in (3, 2, 1, 0)]
        assert n[0] <= n[1] <= n[2] <= n[3]
