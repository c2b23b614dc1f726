"""File-level drop-in: graph documents, DOT export, float WAV.

Parity target: the reference's own graph_io.cpp / wav.cpp compiled into oracle/_ref (with
its JSON library, nlohmann/json, from the image). Documents must have the reference's
layout token for token, every number must denote the same double, and each side must load
the other's documents bit-exactly. (The reference's Grisu2 printer emits a 17-digit form
for ~0.1 % of doubles where a 16-digit one round-trips; the product prints the shortest
form, so the spelling of those few numbers differs while their values are identical.)
WAV files must be byte-identical. Error messages are compared with the reference's.
"""
import os
import re

import numpy as np

import workloads as wl
import pytest

import paper_2408_03204_b200 as mg
from oracle import ref

needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")

TOKEN = re.compile(r'"[^"]*"|[-0-9.eE+]+|[\[\]{}:,]|true|false|null')


def tokens(text):
    out = []
    for tok in TOKEN.findall(text):
        if tok[0] in "-0123456789":
            out.append(("num", float(tok), "." in tok or "e" in tok.lower()))
        else:
            out.append(tok)
    return out


def same_values(a, b):
    assert set(int(k) for k in a) == set(int(k) for k in b)
    for k in a:
        x = np.asarray(a[k], dtype=np.float64)
        y = np.asarray(b[int(k)] if int(k) in b else b[mg.NodeType(int(k))], dtype=np.float64)
        assert x.shape == y.shape
        assert np.array_equal(x.view(np.uint64), y.view(np.uint64)), f"type {k}: values differ"


def console_doc(tracks=2, seed=5):
    g = wl.generate_console(tracks, 0.3, seed)
    P = wl.random_legal_params(mg.to_flat(g).node_types, seed)
    return g, P


@needs_ref
@pytest.mark.parametrize("tracks,seed", [(1, 1), (2, 5), (4, 9)])
def test_graph_to_json_matches_reference_layout(tracks, seed):
    g, P = console_doc(tracks, seed)
    t, e = g.arrays()
    ours = mg.graph_to_json(g, P)
    theirs = ref.graph_to_json(t, e, {int(k): v for k, v in P.items()})
    a, b = tokens(ours), tokens(theirs)
    assert len(a) == len(b)
    assert a == b  # same structure, keys, integers; numbers equal as doubles
    # Layout outside the numbers is identical character for character.
    strip = lambda s: re.sub(r"[-0-9.eE+]+", "#", s)  # noqa: E731
    assert strip(ours) == strip(theirs)


@needs_ref
def test_graph_to_json_without_params_is_byte_identical():
    g = wl.generate_console(3, 0.0, 2)
    t, e = g.arrays()
    assert mg.graph_to_json(g, {}) == ref.graph_to_json(t, e, {})
    empty = mg.Graph()
    assert mg.graph_to_json(empty, {}) == ref.graph_to_json(np.zeros(0, np.int32), np.zeros((0, 4), np.int32), {})


@needs_ref
def test_documents_cross_load_bit_exact(tmp_path):
    g, P = console_doc(3, 11)
    t, e = g.arrays()
    refP = {int(k): v for k, v in P.items()}
    # ours -> reference
    rt, re_, rp = ref.graph_from_json(mg.graph_to_json(g, P))
    assert np.array_equal(rt, t) and np.array_equal(re_, e)
    same_values(P, rp)
    # reference -> ours
    g2, p2 = mg.graph_from_json(ref.graph_to_json(t, e, refP))
    assert g2.node_types == g.node_types and g2.edges == g.edges
    same_values(P, p2)
    # files, both directions
    ref.save_graph(t, e, refP, str(tmp_path / "ref.json"))
    mg.save_graph(g, P, str(tmp_path / "ours.json"))
    g3, p3 = mg.load_graph(str(tmp_path / "ref.json"))
    assert g3.edges == g.edges
    same_values(P, p3)
    _, _, p4 = ref.load_graph(str(tmp_path / "ours.json"))
    same_values(P, p4)


@needs_ref
def test_number_spelling_edge_cases():
    g = mg.Graph()
    a = g.add_node(mg.NodeType.IN)
    b = g.add_node(mg.NodeType.GAIN)
    c = g.add_node(mg.NodeType.OUT)
    g.connect(a, b)
    g.connect(b, c)
    t, e = g.arrays()
    for vals in [(0.0, -0.0), (1e-7, 1e15), (1e16, 123.0), (1e300, 5e-324), (0.0001, 0.00001), (-2.5, 1 / 3),
                 (999999999999999.0, 1234567.125), (2.0 ** 60, -1e-300)]:
        P = {mg.NodeType.GAIN: np.array([vals])}
        ours = mg.graph_to_json(g, P)
        theirs = ref.graph_to_json(t, e, {3: P[mg.NodeType.GAIN]})
        assert ours == theirs, (vals, ours[-120:], theirs[-120:])
        _, back = mg.graph_from_json(ours)
        assert np.array_equal(back[mg.NodeType.GAIN].view(np.uint64), P[mg.NodeType.GAIN].view(np.uint64))


def test_defaults_for_absent_types_and_optional_fields():
    doc = '{"version": 1, "nodes": [{"type": "in"}, {"type": "compressor"}, {"type": "out"}],' \
          ' "edges": [{"src": 0, "dst": 1}, {"src": 1, "dst": 2, "outlet": 0, "inlet": 0}]}'
    g, P = mg.graph_from_json(doc)
    assert g.num_nodes() == 3 and len(g.edges) == 2
    assert np.array_equal(P[mg.NodeType.COMPRESSOR], mg.default_params(g.node_types)[mg.NodeType.COMPRESSOR])


BAD_DOCS = [
    '{"version": 1}',
    '{"nodes": 3}',
    '{"nodes": [{"id": 0}]}',
    '{"nodes": [{"id": 0, "type": "flanger"}]}',
    '{"nodes": [{"id": 1, "type": "in"}]}',
    '{"nodes": [{"type": "in"}, {"type": "out"}], "edges": {"src": 0}}',
    '{"nodes": [{"type": "in"}, {"type": "out"}], "edges": [{"src": 0}]}',
    '{"nodes": [{"type": "in"}, {"type": "gain"}, {"type": "out"}],'
    ' "edges": [{"src": 0, "dst": 1}, {"src": 1, "dst": 2}], "params": {"gain": [[0.0, 0.0], [0.0, 0.0]]}}',
    '{"nodes": [{"type": "in"}, {"type": "eq"}, {"type": "out"}],'
    ' "edges": [{"src": 0, "dst": 1}, {"src": 1, "dst": 2}], "params": {"eq": [[' + ", ".join(["0.0"] * 1000) + ']]}}',
    '{"nodes": [{"type": "in"}, {"type": "out"}], "edges": [{"src": 0, "dst": 1}], "params": {"mix": []}}',
    '{"nodes": [{"type": "in"}, {"type": "out"}], "edges": [{"src": 0, "dst": 1}], "params": {"gain": []}}',
    '{"nodes": [{"type": "in"}, {"type": "out"}], "edges": [{"src": 0, "dst": 1}], "params": {"wah": []}}',
    '{"nodes": [{"type": "in"}, {"type": "out"}], "edges": [{"src": 0, "dst": 1}], "params": []}',
    '{"nodes": [{"type": "in"}, {"type": "gain"}, {"type": "gain"}, {"type": "out"}],'
    ' "edges": [{"src": 0, "dst": 1}, {"src": 1, "dst": 2}, {"src": 2, "dst": 1}, {"src": 2, "dst": 3}]}',
    '{"nodes": [{"type": "in"}, {"type": "out"}], "edges": [{"src": 0, "dst": 1, "outlet": 1}]}',
    '{"nodes": [{"type": "in"}, {"type": "out"}], "edges": [{"src": 0, "dst": 7}]}',
]


@needs_ref
@pytest.mark.parametrize("doc", BAD_DOCS, ids=range(len(BAD_DOCS)))
def test_document_errors_match_reference(doc):
    with pytest.raises(ValueError) as ours:
        mg.graph_from_json(doc)
    with pytest.raises(ValueError) as theirs:
        ref.graph_from_json(doc)
    assert str(ours.value) == str(theirs.value)


@needs_ref
@pytest.mark.parametrize("doc", ['{"nodes": [', 'nope', '{"nodes": [{"type": "in"}]} x', '', '{"a": 1.}'])
def test_parse_errors(doc):
    with pytest.raises(ValueError, match="graph document") as ours:
        mg.graph_from_json(doc)
    with pytest.raises(ValueError, match="graph document"):
        ref.graph_from_json(doc)
    assert "parse error" in str(ours.value)


def test_spec_examples(tmp_path):
    # SPEC.md: unknown type names the tag; eq row of width 1000 -> expected 1024.
    with pytest.raises(ValueError, match="flanger"):
        mg.graph_from_json('{"nodes": [{"type": "flanger"}]}')
    with pytest.raises(ValueError, match="expected 1024"):
        mg.graph_from_json(BAD_DOCS[8])
    with pytest.raises(ValueError, match="cannot open"):
        mg.load_graph(str(tmp_path / "missing.json"))
    g, P = console_doc(2, 3)
    mg.save_graph(g, P, str(tmp_path / "c2.json"))
    g2, P2 = mg.load_graph(str(tmp_path / "c2.json"))
    assert g2.node_types == g.node_types and g2.edges == g.edges
    same_values(P, P2)


@needs_ref
def test_export_dot_matches_reference():
    chain = mg.Graph()
    chain.add_serial_chain([mg.NodeType.IN, mg.NodeType.GAIN, mg.NodeType.OUT])
    for g in [chain, mg.Graph(), wl.generate_console(2, 0.0, 0), wl.generate_console(8, 0.3, 4)]:
        t, e = g.arrays()
        assert mg.export_dot(g) == ref.export_dot(t, e)
    dot = mg.export_dot(chain)
    assert dot.count("[label=") == 3 and dot.count("->") == 2
    assert mg.export_dot(wl.generate_console(2, 0.0, 0)).count("[label=") == 22
    assert mg.export_dot(mg.Graph()) == "digraph {\n  rankdir=LR;\n}\n"


@needs_ref
def test_wav_round_trip_and_byte_identity(tmp_path):
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, size=(1, 2, 1000))
    ours, theirs = str(tmp_path / "ours.wav"), str(tmp_path / "ref.wav")
    mg.write_wav(x, ours, 48000.0)
    ref.write_wav(x, theirs, 48000.0)
    with open(ours, "rb") as f1, open(theirs, "rb") as f2:
        b1, b2 = f1.read(), f2.read()
    assert b1 == b2
    assert b1[0:4] == b"RIFF" and b1[8:12] == b"WAVE"
    y, fs = mg.read_wav(ours)
    assert fs == 48000.0 and y.shape == (1, 2, 1000)
    assert np.array_equal(y, x.astype(np.float32).astype(np.float64))  # bit-exact at float precision
    yr, fsr = ref.read_wav(ours)
    assert fsr == fs and np.array_equal(yr, y)
    # a second round trip is the identity
    mg.write_wav(y, ours, fs)
    assert np.array_equal(mg.read_wav(ours)[0], y)


def _pcm16_wav(path, frames=10):
    import struct
    data = b"\x00\x00" * 2 * frames
    hdr = b"RIFF" + struct.pack("<I", 36 + len(data)) + b"WAVE"
    fmt = b"fmt " + struct.pack("<IHHIIHH", 16, 1, 2, 44100, 44100 * 4, 4, 16)
    with open(path, "wb") as f:
        f.write(hdr + fmt + b"data" + struct.pack("<I", len(data)) + data)


@needs_ref
def test_wav_errors_match_reference(tmp_path):
    p16 = str(tmp_path / "pcm16.wav")
    _pcm16_wav(p16)
    junk = str(tmp_path / "junk.wav")
    with open(junk, "wb") as f:
        f.write(b"not a wave file at all")
    for path in (p16, junk, str(tmp_path / "missing.wav")):
        with pytest.raises(RuntimeError) as ours:
            mg.read_wav(path)
        with pytest.raises(RuntimeError) as theirs:
            ref.read_wav(path)
        assert str(ours.value) == str(theirs.value)
    with pytest.raises(RuntimeError, match="unsupported encoding"):
        mg.read_wav(p16)
    for bad in (np.zeros((2, 2, 8)), np.zeros((1, 1, 8))):
        with pytest.raises(RuntimeError) as ours:
            mg.write_wav(bad, str(tmp_path / "x.wav"))
        with pytest.raises(RuntimeError) as theirs:
            ref.write_wav(bad, str(tmp_path / "y.wav"))
        assert str(ours.value) == str(theirs.value)


def test_wav_render_output_round_trip(tmp_path):
    """A rendered-output-shaped buffer (outputs [1][2][L]) written and re-read as a source."""
    L = 4096
    x = np.stack([mg.uniform_noise(2 * L, 7).reshape(2, L)])
    p = str(tmp_path / "mix.wav")
    mg.write_wav(x, p)
    y, fs = mg.read_wav(p)
    assert fs == 44100.0 and np.array_equal(y, x.astype(np.float32).astype(np.float64))
