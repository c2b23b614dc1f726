"""B200-native batched audio-graph renderer (GRAFX, arXiv 2408.03204) — Python host mirror.

The product is ``libmgb200.so`` (host scheduler in C++ + sm_100a kernels behind the C ABI
declared in ``include/mixgraph_b200.h``). This module binds that ABI with ctypes and mirrors
the reference's C++ render API (``proj/include/mixgraph/{graph,schedule,processors,render}.hpp``)
with the same names, argument meaning and error behaviour: the reference's
``std::invalid_argument`` surfaces here as ``ValueError`` carrying the same message text.

There is no CPU fallback: render/process calls go through CUDA kernels, and importing the
module fails loudly if the shared library is missing.
"""
from __future__ import annotations

import ctypes
import functools
import enum
import os
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmgb200.so")
# Diagnostics only (same-box A/B timing of two builds): load another build of the library.

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(make -C paper_2408_03204_b200/csrc). There is no CPU fallback.")

_lib = ctypes.CDLL(LIB_PATH)

_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_u32 = ctypes.c_uint32
_u64 = ctypes.c_uint64
_dbl = ctypes.c_double
_vp = ctypes.c_void_p
_P = ctypes.POINTER


def _sig(name, restype, *argtypes):
    f = getattr(_lib, name)
    f.restype = restype
    f.argtypes = list(argtypes)
    return f


_sig("mg_last_error", ctypes.c_char_p)
_sig("mg_abi_version", _i32)
_sig("mg_param_width", _i32, _i32)
_sig("mg_graph_validate", _i32, _vp, _i32, _vp, _i32)
_sig("mg_plan_create", _i32, _vp, _i32, _vp, _i32, _i32, _i32, _i32, _P(_vp))
_sig("mg_plan_destroy", None, _vp)
_sig("mg_plan_info", _i32, _vp, _vp)
_sig("mg_plan_type_codes", _i32, _vp, ctypes.c_char_p, _i32)
_sig("mg_plan_subsets", _i32, _vp, _vp, _vp)
_sig("mg_plan_sigma", _i32, _vp, _vp)
_sig("mg_plan_flat", _i32, _vp, _vp, _vp)
_sig("mg_plan_step", _i32, _vp, _i32, _vp, _vp, _vp)
_sig("mg_plan_param_source_rows", _i32, _vp, _i32, _vp)
_sig("mg_plan_reorder_params", _i32, _vp, _vp, _vp, _vp)
_sig("mg_validate_schedule", _i32, _vp, _i32, _vp, _i32, _vp, _i32, _vp, _vp)
_sig("mg_processors_create", _i32, _dbl, _u32, _i32, _dbl, _i32, _P(_vp))
_sig("mg_processors_destroy", None, _vp)
_sig("mg_processors_info", _i32, _vp, _vp)
_sig("mg_render", _i32, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i64, _dbl, _vp, _vp)
_sig("mg_plan_workspace_bytes", _i32, _vp, _vp, _i32, _i64, _P(_u64))
_sig("mg_plan_kernel_count", _i32, _vp, _i32, _i64, _P(_i32))
_sig("mg_plan_step_owners", _i32, _vp, _i32, _i64, _vp)
_sig("mg_plan_shared_pairs", _i32, _vp, _vp, _i32, _i64, _vp)
_sig("mg_plan_fusion_candidates", _i32, _vp, _vp, _vp)
_sig("mg_render_arena", _i32, _vp, _vp, _vp, _vp, _i32, _i64, _vp, _u64, _vp)
_sig("mg_render_arena_profiled", _i32, _vp, _vp, _vp, _vp, _i32, _i64, _vp, _u64, _vp, _vp, _i32)
_sig("mg_profile_steps", _i32, _vp, _vp, _vp, _vp, _i32, _i64, _vp, _u64, _vp, _i32, _vp)
_sig("mg_render_graph_create", _i32, _vp, _vp, _vp, _vp, _i32, _i64, _vp, _u64, _P(_vp))
_sig("mg_render_graph_launch", _i32, _vp, _vp)
_sig("mg_render_graph_destroy", None, _vp)
_sig("mg_pipeline_create", _i32, _vp, _vp, _i32, _i64, _i32, _i32, _i32, _P(_vp))
_sig("mg_pipeline_submit", _i32, _vp, _vp, _vp, _vp, _vp)
_sig("mg_pipeline_sync", _i32, _vp)
_sig("mg_pipeline_destroy", None, _vp)
_sig("mg_backward_workspace_bytes", _i32, _vp, _vp, _i32, _i64, _P(_u64))
_sig("mg_render_backward_arena", _i32, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _i64, _vp, _u64, _vp)
_sig("mg_set_conv_fuse", None, _i32)
_sig("mg_set_dyn_stream", None, _i32)
_sig("mg_set_dyn_pair", None, _i32)
_sig("mg_set_conv_log", None, _i32)
_sig("mg_conv_geometry", _i32, _i64, _i64, _vp)
_sig("mg_set_fft_precision", None, _i32)
_sig("mg_fft_precision", _i32)
_sig("mg_batch_capacity", _i32, _vp, _vp, _i32, _i64, _vp)
_sig("mg_batch_create", _i32, _vp, _i32, _i64, _vp, _i32, _P(_vp))
_sig("mg_batch_submit", _i32, _vp, _vp, _vp, _vp, _i32, _vp, _i32, _i32, _vp)
_sig("mg_batch_sync", _i32, _vp)
_sig("mg_batch_last_arena", _i32, _vp, _P(_vp))
_sig("mg_batch_destroy", None, _vp)
_sig("mg_process", _i32, _vp, _i32, _vp, _vp, _i32, _i32, _i64, _vp, _i32, _i32)
_sig("mg_reverb_kernel", _i32, _vp, _vp, _vp, _vp)
_sig("mg_delay_kernel", _i32, _vp, _vp, _i32, _vp, _vp)
_sig("mg_compressor_gain_log", _dbl, _dbl, _dbl, _dbl, _dbl)
_sig("mg_noisegate_gain_log", _dbl, _dbl, _dbl, _dbl, _dbl)
_sig("mg_check_param_row", _i32, _i32, _vp)
_sig("mg_default_param_row", _i32, _i32, _vp)
_sig("mg_uniform_noise", _i32, _i64, _u32, _vp)
_sig("mg_graph_to_json", _i32, _vp, _i32, _vp, _i32, _vp, _vp, ctypes.c_char_p, _i64, _P(_i64))
_sig("mg_save_graph", _i32, _vp, _i32, _vp, _i32, _vp, _vp, ctypes.c_char_p)
_sig("mg_graph_from_json", _i32, ctypes.c_char_p, _i64, _P(_vp))
_sig("mg_load_graph", _i32, ctypes.c_char_p, _P(_vp))
_sig("mg_doc_info", _i32, _vp, _P(_i32), _P(_i32), _vp)
_sig("mg_doc_graph", _i32, _vp, _vp, _vp)
_sig("mg_doc_params", _i32, _vp, _i32, _vp)
_sig("mg_doc_destroy", None, _vp)
_sig("mg_export_dot", _i32, _vp, _i32, _vp, _i32, ctypes.c_char_p, _i64, _P(_i64))
_sig("mg_write_wav", _i32, _vp, _i32, _i32, _i64, _dbl, ctypes.c_char_p)
_sig("mg_read_wav", _i32, ctypes.c_char_p, _P(_vp))
_sig("mg_audio_info", _i32, _vp, _P(_i64), _P(_dbl))
_sig("mg_audio_samples", _i32, _vp, _vp)
_sig("mg_audio_destroy", None, _vp)


def _check(status: int) -> None:
    if status == 0:
        return
    msg = (_lib.mg_last_error() or b"").decode()
    if status == 1:
        raise ValueError(msg)
    raise RuntimeError(msg)


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(_vp)


class NodeType(enum.IntEnum):
    """`proj/include/mixgraph/types.hpp:12-23`."""
    IN = 0
    OUT = 1
    MIX = 2
    GAIN = 3
    EQ = 4
    COMPRESSOR = 5
    NOISEGATE = 6
    IMAGER = 7
    REVERB = 8
    DELAY = 9


NUM_NODE_TYPES = 10
_CODES = "iomgecnsrd"
_NAMES = ["in", "out", "mix", "gain", "eq", "compressor", "noisegate", "imager", "reverb", "delay"]


def type_code(t: int) -> str:
    return _CODES[int(t)]


def type_name(t: int) -> str:
    return _NAMES[int(t)]


def type_from_code(c: str) -> NodeType:
    return NodeType(_CODES.index(c))


def param_width(t: int) -> int:
    return int(_lib.mg_param_width(int(t)))


class Strategy(enum.IntEnum):
    """`proj/include/mixgraph/schedule.hpp:12-17`."""
    ONE_BY_ONE = 0
    GREEDY = 1
    BEAM = 2
    OPTIMAL = 3


# ---- graph -------------------------------------------------------------------------------

class Graph:
    """Builder (`graph.hpp:26-47`). Edges are (src, dst, outlet, inlet)."""

    def __init__(self):
        self._types: List[int] = []
        self._edges: List[Tuple[int, int, int, int]] = []

    def add_node(self, t: int) -> int:
        self._types.append(int(t))
        return len(self._types) - 1

    def add_serial_chain(self, types: Sequence[int]) -> Tuple[int, int]:
        if not types:
            raise ValueError("add_serial_chain: empty type list")
        first = self.add_node(types[0])
        for t in types[1:]:
            nid = self.add_node(t)
            self.connect(nid - 1, nid)
        return first, len(self._types) - 1

    def connect(self, src: int, dst: int, outlet: int = 0, inlet: int = 0) -> None:
        for nid in (src, dst):
            if nid < 0 or nid >= len(self._types):
                raise ValueError(f"connect: unknown node id {nid}")
        if self._types[dst] == NodeType.IN:
            raise ValueError("connect: in nodes take no incoming edges")
        if self._types[src] == NodeType.OUT:
            raise ValueError("connect: out nodes have no outgoing edges")
        self._edges.append((int(src), int(dst), int(outlet), int(inlet)))

    def validate(self) -> None:
        t, e = self.arrays()
        _check(_lib.mg_graph_validate(_ptr(t), len(t), _ptr(e), len(self._edges)))

    def num_nodes(self) -> int:
        return len(self._types)

    def node_type(self, i: int) -> NodeType:
        return NodeType(self._types[i])

    @property
    def node_types(self) -> List[NodeType]:
        return [NodeType(t) for t in self._types]

    @property
    def edges(self) -> List[Tuple[int, int, int, int]]:
        return list(self._edges)

    def arrays(self) -> Tuple[np.ndarray, np.ndarray]:
        t = np.asarray(self._types, dtype=np.int32)
        e = np.asarray(self._edges, dtype=np.int32).reshape(-1, 4)
        return np.ascontiguousarray(t), np.ascontiguousarray(e)

    @staticmethod
    def from_arrays(types, edges) -> "Graph":
        g = Graph()
        g._types = [int(x) for x in np.asarray(types).reshape(-1)]
        g._edges = [tuple(int(v) for v in row) for row in np.asarray(edges).reshape(-1, 4)]
        return g


def disjoint_union(graphs: Sequence[Graph]) -> Graph:
    """`graph.cpp:116-128`."""
    out = Graph()
    for g in graphs:
        g.validate()
        off = out.num_nodes()
        out._types.extend(g._types)
        out._edges.extend((s + off, d + off, o, i) for (s, d, o, i) in g._edges)
    return out


def default_param_row(t: int) -> np.ndarray:
    row = np.zeros(param_width(t), dtype=np.float64)
    if row.size:
        _check(_lib.mg_default_param_row(int(t), _ptr(row)))
    return row


def default_params(node_types: Sequence[int]) -> Dict[NodeType, np.ndarray]:
    """`graph.cpp:157-169`: one table per parameterised type present, default rows."""
    counts: Dict[int, int] = {}
    for t in node_types:
        if param_width(t) > 0:
            counts[int(t)] = counts.get(int(t), 0) + 1
    return {NodeType(t): np.tile(default_param_row(t), (n, 1)) for t, n in sorted(counts.items())}


def concat_params(stores: Sequence[Dict[NodeType, np.ndarray]]) -> Dict[NodeType, np.ndarray]:
    """`graph.cpp:171-186`."""
    out: Dict[NodeType, np.ndarray] = {}
    for s in stores:
        for t, m in sorted(s.items()):
            if t in out:
                if out[t].shape[1] != m.shape[1]:
                    raise ValueError("concat_params: column mismatch")
                out[t] = np.concatenate([out[t], m], axis=0)
            else:
                out[t] = np.array(m, dtype=np.float64)
    return out


@dataclass
class FlatGraph:
    """`graph.hpp:92-101`."""
    node_types: List[NodeType]
    edges: List[Tuple[int, int, int, int]]
    params: Dict[NodeType, np.ndarray] = field(default_factory=dict)
    num_inputs: int = 0
    num_outputs: int = 0

    def num_nodes(self) -> int:
        return len(self.node_types)

    def arrays(self) -> Tuple[np.ndarray, np.ndarray]:
        return (np.ascontiguousarray(np.asarray([int(t) for t in self.node_types], dtype=np.int32)),
                np.ascontiguousarray(np.asarray(self.edges, dtype=np.int32).reshape(-1, 4)))


def to_flat(g: Graph) -> FlatGraph:
    """`graph.cpp:188-199`: validate, freeze, default parameter rows."""
    g.validate()
    types = g.node_types
    return FlatGraph(types, g.edges, default_params(types),
                     sum(1 for t in types if t == NodeType.IN), sum(1 for t in types if t == NodeType.OUT))


def _tables(params: Dict[int, np.ndarray]):
    """Pointer array [10] + rows [10] for a per-type table dict (keeps arrays alive)."""
    keep = []
    ptrs = (_vp * NUM_NODE_TYPES)()
    rows = np.zeros(NUM_NODE_TYPES, dtype=np.int32)
    for t, m in params.items():
        a = np.ascontiguousarray(m, dtype=np.float64)
        if a.ndim != 2:
            a = a.reshape(-1, param_width(t))
        keep.append(a)
        ptrs[int(t)] = a.ctypes.data
        rows[int(t)] = a.shape[0]
    return ptrs, rows, keep


# ---- scheduling ------------------------------------------------------------------------------

@dataclass
class StepIndex:
    """`schedule.hpp:60-68`."""
    type: NodeType
    gather: List[int]
    aggregate: List[int]
    param_begin: int
    param_end: int
    store_begin: int
    store_end: int


@dataclass
class Schedule:
    type_string: List[NodeType]
    subsets: List[List[int]]

    def num_steps(self) -> int:
        return len(self.subsets) - 1

    def type_codes(self) -> str:
        return "".join(type_code(t) for t in self.type_string)


class RenderData:
    """`schedule.hpp:72-86`, computed by the C++ plan builder (owns the C handle)."""

    def __init__(self, handle, fg: FlatGraph):
        self._h = handle
        self._fg = fg
        info = np.zeros(6, dtype=np.int32)
        _check(_lib.mg_plan_info(self._h, _ptr(info)))
        self.num_steps, self.buffer_rows, self.num_inputs, self.output_begin, self._n_edges, self._n_ts = \
            (int(x) for x in info)

    # The schedule, sigma, flat graph and step table are materialised as Python objects only
    # when asked for (parity tests, inspection); the render path needs just the handle.
    @functools.cached_property
    def schedule(self) -> "Schedule":
        buf = ctypes.create_string_buffer(self._n_ts + 1)
        _check(_lib.mg_plan_type_codes(self._h, buf, self._n_ts + 1))
        sizes = np.zeros(self._n_ts, dtype=np.int32)
        rows = np.zeros(self._fg.num_nodes(), dtype=np.int32)
        _check(_lib.mg_plan_subsets(self._h, _ptr(sizes), _ptr(rows)))
        subsets, off = [], 0
        for sz in sizes:
            subsets.append([int(r) for r in rows[off:off + sz]])
            off += int(sz)
        return Schedule([type_from_code(c) for c in buf.value.decode()], subsets)

    @functools.cached_property
    def sigma(self) -> List[int]:
        sig = np.zeros(self._fg.num_nodes(), dtype=np.int32)
        _check(_lib.mg_plan_sigma(self._h, _ptr(sig)))
        return [int(x) for x in sig]

    @functools.cached_property
    def flat(self) -> "FlatGraph":
        n_edges = self._n_edges
        ft = np.zeros(self._fg.num_nodes(), dtype=np.int32)
        fe = np.zeros((max(n_edges, 1), 4), dtype=np.int32)
        _check(_lib.mg_plan_flat(self._h, _ptr(ft), _ptr(fe)))
        flat = FlatGraph([NodeType(int(t)) for t in ft], [tuple(int(v) for v in r) for r in fe[:n_edges]],
                         {}, self._fg.num_inputs, self._fg.num_outputs)
        if self._fg.params:
            flat.params = self.reorder_params(self._fg.params)
        return flat

    @functools.cached_property
    def steps(self) -> List["StepIndex"]:
        out: List[StepIndex] = []
        head = np.zeros(6, dtype=np.int32)
        for k in range(self.num_steps):
            _check(_lib.mg_plan_step(self._h, k, _ptr(head), None, None))
            g = np.zeros(max(int(head[5]), 1), dtype=np.int32)
            a = np.zeros(max(int(head[5]), 1), dtype=np.int32)
            _check(_lib.mg_plan_step(self._h, k, _ptr(head), _ptr(g), _ptr(a)))
            m = int(head[5])
            out.append(StepIndex(NodeType(int(head[0])), [int(x) for x in g[:m]], [int(x) for x in a[:m]],
                                 int(head[1]), int(head[2]), int(head[3]), int(head[4])))
        return out

    @functools.cached_property
    def param_source_rows(self) -> Dict[NodeType, List[int]]:
        out: Dict[NodeType, List[int]] = {}
        for t in range(NUM_NODE_TYPES):
            n = int(_lib.mg_plan_param_source_rows(self._h, t, None))
            if n > 0:
                rows = np.zeros(n, dtype=np.int32)
                _lib.mg_plan_param_source_rows(self._h, t, _ptr(rows))
                out[NodeType(t)] = [int(x) for x in rows]
        return out

    @property
    def handle(self):
        return self._h

    def reorder_params(self, original: Dict[int, np.ndarray]) -> Dict[NodeType, np.ndarray]:
        """`schedule.cpp:454-471`."""
        ptrs, rows, keep = _tables(original)
        out = {t: np.zeros((len(r), param_width(t)), dtype=np.float64) for t, r in self.param_source_rows.items()}
        optrs = (_vp * NUM_NODE_TYPES)()
        for t, m in out.items():
            optrs[int(t)] = m.ctypes.data
        _check(_lib.mg_plan_reorder_params(self._h, ptrs, _ptr(rows), optrs))
        del keep
        return out

    def original_order(self, render_order: Dict[int, np.ndarray]) -> Dict[NodeType, np.ndarray]:
        """Inverse of reorder_params: per-type tables (e.g. gradients) from render order back
        to the original row order (`schedule.cpp:515-523` param_source_rows)."""
        out = {}
        for t, src in self.param_source_rows.items():
            m = np.asarray(render_order[t])
            o = np.empty_like(m)
            o[np.asarray(src, dtype=np.int64)] = m
            out[NodeType(t)] = o
        return out

    def kernel_count(self, batch: int, length: int) -> int:
        c = _i32()
        _check(_lib.mg_plan_kernel_count(self._h, batch, length, ctypes.byref(c)))
        return int(c.value)

    def shared_pairs(self, procs: "ProcessorSet", batch: int, length: int) -> np.ndarray:
        """pairs[k] = slots of step k reusing a signal spectrum of step k-1 in a render with
        these processors / batch / length (adjacent delay / reverb sends of the same tracks);
        mg_plan_shared_pairs."""
        out = np.zeros(self.num_steps, dtype=np.int32)
        _check(_lib.mg_plan_shared_pairs(self._h, procs.handle, batch, length, out.ctypes.data_as(_vp)))
        return out

    def fusion_candidates(self):
        """Host-side plan analysis (mg_plan_fusion_candidates): (share_pairs, reads_prev_rows),
        per step — slots pairing with the previous conv step on a common source row, and
        whether the step reads exactly the previous step's rows slot by slot."""
        a = np.zeros(self.num_steps, dtype=np.int32)
        b = np.zeros(self.num_steps, dtype=np.int32)
        _check(_lib.mg_plan_fusion_candidates(self._h, a.ctypes.data_as(_vp), b.ctypes.data_as(_vp)))
        return a, b.astype(bool)

    def step_owners(self, batch: int, length: int) -> np.ndarray:
        """owner[k] = the step whose kernel launch computes step k (itself, the head of a fused
        pointwise run, or the producer whose epilogue computes it); mg_plan_step_owners."""
        out = np.zeros(self.num_steps, dtype=np.int32)
        _check(_lib.mg_plan_step_owners(self._h, batch, length, out.ctypes.data_as(_vp)))
        return out

    def __del__(self, _destroy=_lib.mg_plan_destroy):
        h, self._h = getattr(self, "_h", None), None
        if h:
            _destroy(h)


def compute_render_data(fg: FlatGraph, strategy: int = Strategy.GREEDY, beam_width: int = 32,
                        optimal_node_cap: int = 256) -> RenderData:
    """`schedule.cpp:473-525` (validates the graph like to_flat)."""
    t, e = fg.arrays()
    h = _vp()
    _check(_lib.mg_plan_create(_ptr(t), len(t), _ptr(e), len(fg.edges), int(strategy), int(beam_width),
                               int(optimal_node_cap), ctypes.byref(h)))
    return RenderData(h, fg)


class _ArrayGraph:
    """Minimal FlatGraph stand-in over (types, edges) int32 arrays (no Python node lists)."""

    def __init__(self, types: np.ndarray, edges: np.ndarray):
        self._t = np.ascontiguousarray(types, dtype=np.int32)
        self._e = np.ascontiguousarray(np.asarray(edges, dtype=np.int32).reshape(-1, 4))
        self.params: Dict[NodeType, np.ndarray] = {}
        self.num_inputs = int(np.count_nonzero(self._t == int(NodeType.IN)))
        self.num_outputs = int(np.count_nonzero(self._t == int(NodeType.OUT)))

    def num_nodes(self) -> int:
        return len(self._t)

    def arrays(self) -> Tuple[np.ndarray, np.ndarray]:
        return self._t, self._e


def compute_render_data_arrays(types: np.ndarray, edges: np.ndarray, strategy: int = Strategy.GREEDY,
                               beam_width: int = 32, optimal_node_cap: int = 256) -> RenderData:
    """compute_render_data straight from int32 arrays (types [V], edges [E, 4]) — the fast
    path for large unions whose topology changes every batch (no Python graph objects)."""
    ag = _ArrayGraph(types, edges)
    t, e = ag.arrays()
    h = _vp()
    _check(_lib.mg_plan_create(_ptr(t), len(t), _ptr(e), len(e), int(strategy), int(beam_width),
                               int(optimal_node_cap), ctypes.byref(h)))
    return RenderData(h, ag)


def make_schedule(fg: FlatGraph, strategy: int = Strategy.GREEDY, beam_width: int = 32,
                  optimal_node_cap: int = 256) -> Schedule:
    """`schedule.cpp:325-338` (returned from the full plan build)."""
    return compute_render_data(fg, strategy, beam_width, optimal_node_cap).schedule


def validate_schedule(fg: FlatGraph, s: Schedule) -> None:
    """`schedule.cpp:351-395`."""
    t, e = fg.arrays()
    ts = np.asarray([int(x) for x in s.type_string], dtype=np.int32)
    sizes = np.asarray([len(x) for x in s.subsets], dtype=np.int32)
    rows = np.asarray([r for x in s.subsets for r in x] or [0], dtype=np.int32)
    _check(_lib.mg_validate_schedule(_ptr(t), len(t), _ptr(e), len(fg.edges), _ptr(ts), len(ts), _ptr(sizes), _ptr(rows)))


# ---- processors and rendering -----------------------------------------------------------------

class ProcessorSet:
    """`processors.hpp:25-66` with device-resident constants on CUDA device `device`."""

    def __init__(self, sample_rate: float = 44100.0, reverb_seed: int = 0, envelope_taps: int = 32768,
                 energy_floor: float = 1e-7, device: int = 0):
        self._h = _vp()
        _check(_lib.mg_processors_create(float(sample_rate), int(reverb_seed), int(envelope_taps), float(energy_floor),
                                         int(device), ctypes.byref(self._h)))
        info = np.zeros(3, dtype=np.int64)
        _check(_lib.mg_processors_info(self._h, _ptr(info)))
        self.sample_rate = float(sample_rate)
        self.device = int(device)
        self.delay_span, self.delay_window, self.reverb_length = (int(x) for x in info)

    @property
    def handle(self):
        return self._h

    def process(self, t: int, inp: np.ndarray, slots: int, batch: int, length: int,
                params: Optional[np.ndarray] = None, param_offset: int = 0) -> np.ndarray:
        """`processors.cpp:229-282`: inp [slots][batch][2][length] -> same shape."""
        x = np.ascontiguousarray(inp, dtype=np.float64)
        out = np.zeros_like(x)
        p = None if params is None else np.ascontiguousarray(params, dtype=np.float64).reshape(-1, param_width(t))
        _check(_lib.mg_process(self._h, int(t), _ptr(x), _ptr(out), slots, batch, length, _ptr(p),
                               0 if p is None else p.shape[0], param_offset))
        return out

    def process_node(self, t: int, inp: np.ndarray, params: Sequence[float] = ()) -> np.ndarray:
        """`processors.cpp:284-297`: inp [batch][2][length]."""
        x = np.asarray(inp, dtype=np.float64)
        if x.ndim != 3 or x.shape[1] != 2:
            raise ValueError("process_node: processors are stereo (2 channels)")
        p = np.asarray(params, dtype=np.float64).reshape(-1)
        if p.size != param_width(t):
            raise ValueError(f"{type_name(t)}: expected {param_width(t)} parameters")
        return self.process(t, x[None], 1, x.shape[0], x.shape[2], p.reshape(1, -1) if p.size else None, 0)[0]

    def reverb_kernel(self, row: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
        r = np.ascontiguousarray(row, dtype=np.float64)
        left = np.zeros(self.reverb_length)
        right = np.zeros(self.reverb_length)
        _check(_lib.mg_reverb_kernel(self._h, _ptr(r), _ptr(left), _ptr(right)))
        return left, right

    def delay_kernel(self, row: np.ndarray, channel: int) -> np.ndarray:
        r = np.ascontiguousarray(row, dtype=np.float64)
        k = np.zeros(self.delay_span)
        _check(_lib.mg_delay_kernel(self._h, _ptr(r), int(channel), _ptr(k), None))
        return k

    def delay_positions(self, row: np.ndarray, channel: int) -> List[int]:
        r = np.ascontiguousarray(row, dtype=np.float64)
        pos = np.zeros(20, dtype=np.int64)
        _check(_lib.mg_delay_kernel(self._h, _ptr(r), int(channel), None, _ptr(pos)))
        return [int(x) for x in pos]

    def __del__(self, _destroy=_lib.mg_processors_destroy):
        h, self._h = getattr(self, "_h", None), None
        if h:
            _destroy(h)


def compressor_gain_log(g_u, threshold, knee, ratio) -> float:
    return float(_lib.mg_compressor_gain_log(g_u, threshold, knee, ratio))


def noisegate_gain_log(g_u, threshold, knee, ratio) -> float:
    return float(_lib.mg_noisegate_gain_log(g_u, threshold, knee, ratio))


def check_param_row(t: int, row: Sequence[float]) -> None:
    r = np.ascontiguousarray(row, dtype=np.float64)
    _check(_lib.mg_check_param_row(int(t), _ptr(r)))


def render(rd: RenderData, procs: ProcessorSet, params: Optional[Dict[int, np.ndarray]], sources: np.ndarray,
           keep_intermediates: bool = False, sample_rate: Optional[float] = None, out: Optional[np.ndarray] = None):
    """`render.cpp:14-81`. sources [K][B][2][L] (host, double); params in render order
    (RenderData.reorder_params) or None for rd.flat.params. Returns outputs
    [num_outputs][B][2][L] (and intermediates [rows][B][2][L], original row order)."""
    src = np.ascontiguousarray(sources, dtype=np.float64)
    if src.ndim != 4:
        raise ValueError("render: sources must be [K][B][2][L]")
    if src.shape[0] != rd.num_inputs:
        raise ValueError(f"render: expected {rd.num_inputs} sources, got {src.shape[0]}")
    if src.shape[2] != 2:
        raise ValueError("render: sources must be stereo")
    k, b, _, n = src.shape
    ptrs, rows, keep = _tables(rd.flat.params if params is None else params)
    shape = (rd.buffer_rows - rd.output_begin, b, 2, n)
    if out is not None:
        if out.shape != shape or out.dtype != np.float64 or not out.flags.c_contiguous:
            raise ValueError(f"render: out must be a contiguous float64 array of shape {shape}")
        outs = out
    else:
        outs = np.zeros(shape)
    inter = np.zeros((rd.buffer_rows, b, 2, n)) if keep_intermediates else None
    fs = procs.sample_rate if sample_rate is None else sample_rate
    _check(_lib.mg_render(rd.handle, procs.handle, ptrs, _ptr(rows), _ptr(src), k, b, n, fs, _ptr(outs), _ptr(inter)))
    del keep
    return (outs, inter) if keep_intermediates else outs


def set_conv_fuse(mode: int) -> None:
    """mg_set_conv_fuse: -1 auto (default), 0 separate kernel-spectrum rows pass, 1 fused."""
    _lib.mg_set_conv_fuse(int(mode))


def set_dyn_stream(mode: int) -> None:
    """mg_set_dyn_stream: -1 auto (default), 0 chained look-back scan, 1 streaming scan
    (one CTA per sequence) wherever legal."""
    _lib.mg_set_dyn_stream(int(mode))


def set_dyn_pair(mode: int) -> None:
    """mg_set_dyn_pair: a compressor / noisegate step followed by one reading exactly its rows
    runs as one streaming kernel (-1 / 1, default) or two (0)."""
    _lib.mg_set_dyn_pair(int(mode))


def conv_geometry(length: int, taps: int) -> Dict[str, int]:
    """mg_conv_geometry: the segmented overlap-save transform a long convolution uses."""
    out = np.zeros(5, dtype=np.int64)
    _check(_lib.mg_conv_geometry(int(length), int(taps), out.ctypes.data_as(_vp)))
    return dict(zip(("log_n", "log_n1", "log_n2", "nseg", "seg"), (int(x) for x in out)))


def set_fft_precision(bits: int) -> None:
    """mg_set_fft_precision: arithmetic of the FFT-based steps, 32 or 64 bits (arena fp32)."""
    _lib.mg_set_fft_precision(int(bits))


def fft_precision() -> int:
    return int(_lib.mg_fft_precision())


def set_conv_log(log_n: int) -> None:
    """mg_set_conv_log: 0 automatic segment size (default), 13..22 forces 2^log_n-point segments."""
    _lib.mg_set_conv_log(int(log_n))


def uniform_noise(n: int, seed: int) -> np.ndarray:
    """`dsp.cpp:222-230`."""
    out = np.zeros(n)
    _check(_lib.mg_uniform_noise(n, seed, _ptr(out)))
    return out


from .device import BatchRenderer, DeviceRenderer, RenderPipeline  # noqa: E402  (torch-backed device path)

__all__ = [
    "NodeType", "Strategy", "Graph", "FlatGraph", "RenderData", "StepIndex", "Schedule", "ProcessorSet",
    "BatchRenderer", "DeviceRenderer", "RenderPipeline", "to_flat", "disjoint_union", "compute_render_data_arrays",
    "default_params", "default_param_row", "concat_params",
    "compute_render_data", "make_schedule", "validate_schedule", "render", "param_width", "type_code", "type_name",
    "uniform_noise", "compressor_gain_log", "noisegate_gain_log",
    "check_param_row", "LIB_PATH",
]


# ---- file-level I/O (graph_io.hpp:20-28, wav.hpp:11-12) -------------------------------------

def _text_call(fn, *args) -> str:
    n = ctypes.c_int64()
    _check(fn(*args, None, 0, ctypes.byref(n)))
    buf = ctypes.create_string_buffer(n.value + 1)
    _check(fn(*args, buf, n.value + 1, ctypes.byref(n)))
    return buf.raw[: n.value].decode()


def graph_to_json(g: Graph, params: Optional[Dict[int, np.ndarray]] = None) -> str:
    """`graph_io.cpp:19-49`: sorted keys, two-space indent, shortest round-trip numbers."""
    t, e = g.arrays()
    ptrs, rows, _keep = _tables(params or {})
    return _text_call(_lib.mg_graph_to_json, _ptr(t), len(t), _ptr(e), len(e), ptrs, _ptr(rows))


def _doc_out(h) -> Tuple[Graph, Dict[NodeType, np.ndarray]]:
    try:
        nn, ne = _i32(), _i32()
        rows = np.zeros(NUM_NODE_TYPES, dtype=np.int32)
        _check(_lib.mg_doc_info(h, ctypes.byref(nn), ctypes.byref(ne), _ptr(rows)))
        t = np.zeros(nn.value, dtype=np.int32)
        e = np.zeros((ne.value, 4), dtype=np.int32)
        _check(_lib.mg_doc_graph(h, _ptr(t), _ptr(e)))
        params: Dict[NodeType, np.ndarray] = {}
        for ti in range(NUM_NODE_TYPES):
            if rows[ti] >= 0:
                m = np.zeros((int(rows[ti]), param_width(ti)), dtype=np.float64)
                _check(_lib.mg_doc_params(h, ti, _ptr(m)))
                params[NodeType(ti)] = m
        return Graph.from_arrays(t, e), params
    finally:
        _lib.mg_doc_destroy(h)


def graph_from_json(text: str) -> Tuple[Graph, Dict[NodeType, np.ndarray]]:
    """`graph_io.cpp:51-117`: validated graph + parameter tables (defaults where absent)."""
    raw = text.encode()
    h = _vp()
    _check(_lib.mg_graph_from_json(raw, len(raw), ctypes.byref(h)))
    return _doc_out(h)


def save_graph(g: Graph, params: Optional[Dict[int, np.ndarray]], path: str) -> None:
    """`graph_io.cpp:119-124`."""
    t, e = g.arrays()
    ptrs, rows, _keep = _tables(params or {})
    _check(_lib.mg_save_graph(_ptr(t), len(t), _ptr(e), len(e), ptrs, _ptr(rows), os.fsencode(path)))


def load_graph(path: str) -> Tuple[Graph, Dict[NodeType, np.ndarray]]:
    """`graph_io.cpp:126-132`."""
    h = _vp()
    _check(_lib.mg_load_graph(os.fsencode(path), ctypes.byref(h)))
    return _doc_out(h)


def export_dot(g: Graph) -> str:
    """`graph_io.cpp:134-143`: deterministic DOT, nodes labelled with their letter code."""
    t, e = g.arrays()
    return _text_call(_lib.mg_export_dot, _ptr(t), len(t), _ptr(e), len(e))


def write_wav(samples: np.ndarray, path: str, sample_rate: float = 44100.0) -> None:
    """`wav.cpp:39-83`: samples [1][2][L] (or [2][L]) as 32-bit float stereo PCM."""
    a = np.ascontiguousarray(samples, dtype=np.float64)
    if a.ndim == 2:
        a = a[None]
    if a.ndim != 3:
        raise ValueError("write_wav: samples must be [batch][channels][length]")
    _check(_lib.mg_write_wav(_ptr(a), a.shape[0], a.shape[1], a.shape[2], float(sample_rate), os.fsencode(path)))


def read_wav(path: str) -> Tuple[np.ndarray, float]:
    """`wav.cpp:85-133` -> (samples [1][2][L] float64, sample rate)."""
    h = _vp()
    _check(_lib.mg_read_wav(os.fsencode(path), ctypes.byref(h)))
    try:
        n, fs = ctypes.c_int64(), ctypes.c_double()
        _check(_lib.mg_audio_info(h, ctypes.byref(n), ctypes.byref(fs)))
        out = np.zeros((1, 2, n.value), dtype=np.float64)
        _check(_lib.mg_audio_samples(h, _ptr(out)))
        return out, fs.value
    finally:
        _lib.mg_audio_destroy(h)
