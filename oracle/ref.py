"""ORACLE — test infrastructure only (tests/, __graft_entry__.smoke(), bench.py cpu_baseline).

ctypes access to the UNMODIFIED reference compiled by oracle/Makefile into
oracle/_ref/libmixgraph_ref.so (reference sources from /root/reference/proj + the
FFTW/doctest stand-ins in oracle/shim/; entry points in oracle/ref_capi.cpp). Nothing in
the product imports this module. Parameter tables are dicts {node type: [rows][width]}
in ORIGINAL node order; audio is [K][B][2][L] float64.
"""
from __future__ import annotations

import ctypes
import os
from typing import Dict, List, Optional, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(_HERE, "_ref", "libmixgraph_ref.so")
WIDTHS = [0, 0, 0, 2, 1024, 4, 4, 1, 768, 880]
_vp = ctypes.c_void_p
_i32, _i64, _u32, _dbl = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_double


def available() -> bool:
    return os.path.exists(REF_SO)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{REF_SO} not built (make -C oracle)")
        L = ctypes.CDLL(REF_SO)

        def sig(name, res, *args):
            f = getattr(L, name)
            f.restype = res
            f.argtypes = list(args)

        sig("ref_last_error", ctypes.c_char_p)
        sig("ref_console", _i32, _i32, _dbl, _u32, _vp, _i32, _vp, _i32, _vp, _vp)
        sig("ref_random_dag", _i32, _u32, _i32, _i32, _i32, _vp, _i32, _vp, _i32, _vp, _vp)
        sig("ref_four_track_snippet", _i32, _vp, _i32, _vp, _i32, _vp, _vp)
        sig("ref_random_legal_params", _i32, _vp, _i32, _vp, _i32, _u32, _vp)
        sig("ref_default_param_row", _i32, _i32, _vp)
        sig("ref_plan_create", _i32, _vp, _i32, _vp, _i32, _i32, _i32, _i32, ctypes.POINTER(_vp))
        sig("ref_plan_destroy", None, _vp)
        sig("ref_plan_info", _i32, _vp, _vp)
        sig("ref_plan_type_codes", _i32, _vp, ctypes.c_char_p, _i32)
        sig("ref_plan_subsets", _i32, _vp, _vp, _vp)
        sig("ref_plan_sigma", _i32, _vp, _vp)
        sig("ref_plan_flat", _i32, _vp, _vp, _vp)
        sig("ref_plan_step", _i32, _vp, _i32, _vp, _vp, _vp)
        sig("ref_plan_param_source_rows", _i32, _vp, _i32, _vp)
        sig("ref_render", _i32, _vp, _dbl, _u32, _i32, _dbl, _vp, _vp, _vp, _i32, _i64, _vp, _vp)
        sig("ref_render_parallel", _i32, _vp, _dbl, _u32, _i32, _dbl, _vp, _vp, _vp, _i32, _i64, _i32, _vp, _i32,
            _vp, _vp, _i32, _dbl)
        sig("ref_render_reference", _i32, _vp, _i32, _vp, _i32, _dbl, _u32, _i32, _dbl, _vp, _vp, _vp, _i32, _i64, _vp)
        sig("ref_process", _i32, _i32, _vp, _vp, _i32, _i32, _i64, _vp, _i32, _i32, _dbl, _u32, _i32, _dbl)
        sig("ref_reverb_kernel", _i32, _dbl, _u32, _vp, _vp, _vp, ctypes.POINTER(_i64))
        sig("ref_delay_kernel", _i32, _dbl, _vp, _i32, _vp, _vp, ctypes.POINTER(_i64))
        sig("ref_zero_phase_fir", _i32, _vp, _i32, _vp)
        sig("ref_uniform_noise", _i32, _i64, _u32, _vp)
        sig("ref_fit", _i32, _vp, _i32, _vp, _i32, _dbl, _vp, _vp, _vp, _vp, _vp, _i32, _i64, _vp, _i32, _i32, _dbl,
            _dbl, _vp)
        sig("ref_graph_to_json", _i32, _vp, _i32, _vp, _i32, _vp, _vp, ctypes.c_char_p, _i64, ctypes.POINTER(_i64))
        sig("ref_save_graph", _i32, _vp, _i32, _vp, _i32, _vp, _vp, ctypes.c_char_p)
        sig("ref_graph_from_json", _i32, ctypes.c_char_p, ctypes.POINTER(_vp))
        sig("ref_load_graph", _i32, ctypes.c_char_p, ctypes.POINTER(_vp))
        sig("ref_doc_info", _i32, _vp, ctypes.POINTER(_i32), ctypes.POINTER(_i32), _vp)
        sig("ref_doc_graph", _i32, _vp, _vp, _vp)
        sig("ref_doc_params", _i32, _vp, _i32, _vp)
        sig("ref_doc_destroy", None, _vp)
        sig("ref_export_dot", _i32, _vp, _i32, _vp, _i32, ctypes.c_char_p, _i64, ctypes.POINTER(_i64))
        sig("ref_write_wav", _i32, _vp, _i32, _i32, _i64, _dbl, ctypes.c_char_p)
        sig("ref_read_wav", _i32, ctypes.c_char_p, _vp, _i64, ctypes.POINTER(_i64), ctypes.POINTER(_dbl))
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(_vp)


def _check(st):
    if st != 0:
        msg = (lib().ref_last_error() or b"").decode()
        raise (ValueError if st == 1 else RuntimeError)(msg)


def _graph_out(fn, *args, cap_nodes=200000, cap_edges=400000):
    t = np.zeros(cap_nodes, dtype=np.int32)
    e = np.zeros((cap_edges, 4), dtype=np.int32)
    nn, ne = _i32(), _i32()
    _check(fn(*args, _p(t), cap_nodes, _p(e), cap_edges, ctypes.byref(nn), ctypes.byref(ne)))
    return t[: nn.value].copy(), e[: ne.value].copy()


def console(tracks: int, prune: float = 0.0, seed: int = 0) -> Tuple[np.ndarray, np.ndarray]:
    """console.cpp:10-44 -> (node types, edges[E][4])."""
    return _graph_out(lib().ref_console, tracks, prune, seed)


def random_dag(seed: int, min_nodes: int, max_nodes: int, heavy: bool = True):
    """tests/support/test_util.cpp:17-61 with a fresh mt19937(seed)."""
    return _graph_out(lib().ref_random_dag, seed, min_nodes, max_nodes, int(heavy))


def four_track_snippet():
    return _graph_out(lib().ref_four_track_snippet)


def _table_ptrs(tables: Dict[int, np.ndarray]):
    ptrs = (_vp * 10)()
    rows = np.zeros(10, dtype=np.int32)
    keep = []
    for t, m in tables.items():
        a = np.ascontiguousarray(m, dtype=np.float64).reshape(-1, WIDTHS[int(t)])
        keep.append(a)
        ptrs[int(t)] = a.ctypes.data
        rows[int(t)] = a.shape[0]
    return ptrs, rows, keep


def random_legal_params(types, edges, seed: int) -> Dict[int, np.ndarray]:
    types = np.ascontiguousarray(types, dtype=np.int32)
    edges = np.ascontiguousarray(edges, dtype=np.int32).reshape(-1, 4)
    counts: Dict[int, int] = {}
    for t in types:
        if WIDTHS[int(t)]:
            counts[int(t)] = counts.get(int(t), 0) + 1
    out = {t: np.zeros((n, WIDTHS[t])) for t, n in sorted(counts.items())}
    ptrs = (_vp * 10)()
    for t, m in out.items():
        ptrs[t] = m.ctypes.data
    _check(lib().ref_random_legal_params(_p(types), len(types), _p(edges), len(edges), seed, ptrs))
    return out


def uniform_noise(n: int, seed: int) -> np.ndarray:
    out = np.zeros(n)
    _check(lib().ref_uniform_noise(n, seed, _p(out)))
    return out


class Plan:
    """compute_render_data (schedule.cpp:473-525) of the reference."""

    def __init__(self, types, edges, strategy: int = 1, beam_width: int = 32, optimal_cap: int = 256):
        self.types = np.ascontiguousarray(types, dtype=np.int32)
        self.edges = np.ascontiguousarray(edges, dtype=np.int32).reshape(-1, 4)
        self.h = _vp()
        _check(lib().ref_plan_create(_p(self.types), len(self.types), _p(self.edges), len(self.edges), strategy,
                                     beam_width, optimal_cap, ctypes.byref(self.h)))
        info = np.zeros(6, dtype=np.int32)
        lib().ref_plan_info(self.h, _p(info))
        self.num_steps, self.buffer_rows, self.num_inputs, self.output_begin, ne, nts = (int(x) for x in info)
        buf = ctypes.create_string_buffer(nts + 1)
        lib().ref_plan_type_codes(self.h, buf, nts + 1)
        self.type_codes = buf.value.decode()
        sizes = np.zeros(nts, dtype=np.int32)
        rows = np.zeros(len(self.types), dtype=np.int32)
        lib().ref_plan_subsets(self.h, _p(sizes), _p(rows))
        self.subsets, off = [], 0
        for s in sizes:
            self.subsets.append([int(r) for r in rows[off:off + s]])
            off += int(s)
        sig = np.zeros(len(self.types), dtype=np.int32)
        lib().ref_plan_sigma(self.h, _p(sig))
        self.sigma = [int(x) for x in sig]
        ft = np.zeros(len(self.types), dtype=np.int32)
        fe = np.zeros((max(ne, 1), 4), dtype=np.int32)
        lib().ref_plan_flat(self.h, _p(ft), _p(fe))
        self.flat_types = [int(x) for x in ft]
        self.flat_edges = [tuple(int(v) for v in r) for r in fe[:ne]]
        self.steps = []
        head = np.zeros(6, dtype=np.int32)
        for k in range(self.num_steps):
            lib().ref_plan_step(self.h, k, _p(head), None, None)
            m = int(head[5])
            g = np.zeros(max(m, 1), dtype=np.int32)
            a = np.zeros(max(m, 1), dtype=np.int32)
            lib().ref_plan_step(self.h, k, _p(head), _p(g), _p(a))
            self.steps.append(dict(type=int(head[0]), param_begin=int(head[1]), param_end=int(head[2]),
                                   store_begin=int(head[3]), store_end=int(head[4]),
                                   gather=[int(x) for x in g[:m]], aggregate=[int(x) for x in a[:m]]))
        self.param_source_rows = {}
        for t in range(10):
            n = lib().ref_plan_param_source_rows(self.h, t, None)
            if n > 0:
                out = np.zeros(n, dtype=np.int32)
                lib().ref_plan_param_source_rows(self.h, t, _p(out))
                self.param_source_rows[t] = [int(x) for x in out]

    def render(self, params: Dict[int, np.ndarray], sources: np.ndarray, sample_rate: float = 44100.0,
               reverb_seed: int = 0, envelope_taps: int = 32768, energy_floor: float = 1e-7,
               keep_intermediates: bool = False):
        """render.cpp:14-81 with rd.reorder_params(params) (params in ORIGINAL row order)."""
        src = np.ascontiguousarray(sources, dtype=np.float64)
        k, b, _, n = src.shape
        ptrs, rows, keep = _table_ptrs(params)
        outs = np.zeros((self.buffer_rows - self.output_begin, b, 2, n))
        inter = np.zeros((self.buffer_rows, b, 2, n)) if keep_intermediates else None
        _check(lib().ref_render(self.h, sample_rate, reverb_seed, envelope_taps, energy_floor, ptrs, _p(rows), _p(src),
                                b, n, _p(outs), _p(inter)))
        return (outs, inter) if keep_intermediates else outs

    def render_parallel(self, params: Dict[int, np.ndarray], sources: np.ndarray, sample_rate: float = 44100.0,
                        threads: Optional[int] = None, keep=None, reverb_seed: int = 0, envelope_taps: int = 32768,
                        energy_floor: float = 1e-7, round_f32: bool = False, perturb: float = 0.0):
        """render.cpp:14-81 with each step's slots on `threads` host threads (ref_render_parallel:
        the reference's own gather order and ProcessorSet::process per slot; rows freed after
        their last reader). Returns outputs, or (outputs, kept) with kept[j] = the row of
        ORIGINAL node keep[j] (as render()'s intermediates). round_f32 (diagnostic): rows rounded
        to float between steps (the reference's arithmetic over an fp32 arena). perturb > 0
        (conditioning probe): uniform noise of amplitude perturb * row peak added to every
        processed row (the global per-step error of an FFT-based fp32 renderer)."""
        import os
        src = np.ascontiguousarray(sources, dtype=np.float64)
        k, b, _, n = src.shape
        ptrs, rows, _keep = _table_ptrs(params)
        outs = np.zeros((self.buffer_rows - self.output_begin, b, 2, n))
        kk = None if keep is None else np.ascontiguousarray(keep, dtype=np.int32)
        kept = None if kk is None else np.zeros((len(kk), b, 2, n))
        _check(lib().ref_render_parallel(self.h, sample_rate, reverb_seed, envelope_taps, energy_floor, ptrs, _p(rows),
                                         _p(src), b, n, int(threads or os.cpu_count() or 1), _p(kk),
                                         0 if kk is None else len(kk), _p(outs), _p(kept), int(bool(round_f32)),
                                         float(perturb)))
        return outs if kk is None else (outs, kept)

    def __del__(self):
        h, self.h = getattr(self, "h", None), None
        if h and _lib is not None:
            try:
                _lib.ref_plan_destroy(h)
            except Exception:
                pass


def render_reference(types, edges, params, sources, sample_rate=44100.0, reverb_seed=0, envelope_taps=32768,
                     energy_floor=1e-7) -> np.ndarray:
    """reference.cpp:155-328 (per-node direct-convolution oracle; small sizes only)."""
    types = np.ascontiguousarray(types, dtype=np.int32)
    edges = np.ascontiguousarray(edges, dtype=np.int32).reshape(-1, 4)
    src = np.ascontiguousarray(sources, dtype=np.float64)
    k, b, _, n = src.shape
    n_out = int(np.sum(types == 1))
    ptrs, rows, keep = _table_ptrs(params)
    outs = np.zeros((n_out, b, 2, n))
    _check(lib().ref_render_reference(_p(types), len(types), _p(edges), len(edges), sample_rate, reverb_seed,
                                      envelope_taps, energy_floor, ptrs, _p(rows), _p(src), b, n, _p(outs)))
    return outs


def process(t: int, inp: np.ndarray, slots: int, batch: int, length: int, params: Optional[np.ndarray] = None,
            param_offset: int = 0, sample_rate: float = 44100.0, reverb_seed: int = 0, envelope_taps: int = 32768,
            energy_floor: float = 1e-7) -> np.ndarray:
    """processors.cpp:229-282."""
    x = np.ascontiguousarray(inp, dtype=np.float64)
    out = np.zeros_like(x)
    p = None if params is None else np.ascontiguousarray(params, dtype=np.float64).reshape(-1, WIDTHS[t])
    _check(lib().ref_process(t, _p(x), _p(out), slots, batch, length, _p(p), 0 if p is None else p.shape[0],
                             param_offset, sample_rate, reverb_seed, envelope_taps, energy_floor))
    return out


def reverb_kernel(row: np.ndarray, sample_rate: float = 44100.0, reverb_seed: int = 0):
    r = np.ascontiguousarray(row, dtype=np.float64)
    n = _i64()
    _check(lib().ref_reverb_kernel(sample_rate, reverb_seed, _p(r), None, None, ctypes.byref(n)))
    left, right = np.zeros(n.value), np.zeros(n.value)
    _check(lib().ref_reverb_kernel(sample_rate, reverb_seed, _p(r), _p(left), _p(right), ctypes.byref(n)))
    return left, right


def delay_kernel(row: np.ndarray, channel: int, sample_rate: float = 44100.0):
    r = np.ascontiguousarray(row, dtype=np.float64)
    span = _i64()
    _check(lib().ref_delay_kernel(sample_rate, _p(r), channel, None, None, ctypes.byref(span)))
    k = np.zeros(span.value)
    pos = np.zeros(20, dtype=np.int64)
    _check(lib().ref_delay_kernel(sample_rate, _p(r), channel, _p(k), _p(pos), ctypes.byref(span)))
    return k, [int(x) for x in pos]


def fit(types, edges, params, sources, target, trainable, steps: int, learning_rate: float, fd_step: float = 1e-3,
        sample_rate: float = 44100.0):
    """fit.cpp:25-96 (central differences + gradient descent). Returns (params, loss_history)."""
    types = np.ascontiguousarray(types, dtype=np.int32)
    edges = np.ascontiguousarray(edges, dtype=np.int32).reshape(-1, 4)
    src = np.ascontiguousarray(sources, dtype=np.float64)
    tgt = np.ascontiguousarray(target, dtype=np.float64)
    k, b, _, n = src.shape
    ptrs, rows, keep = _table_ptrs(params)
    out = {t: np.array(v, dtype=np.float64, copy=True) for t, v in params.items()}
    optrs, _, keep2 = _table_ptrs(out)
    tr = np.ascontiguousarray([int(t) for t in trainable], dtype=np.int32)
    hist = np.zeros(steps + 1)
    _check(lib().ref_fit(_p(types), len(types), _p(edges), len(edges), sample_rate, ptrs, _p(rows), optrs, _p(src),
                         _p(tgt), b, n, _p(tr), len(tr), steps, learning_rate, fd_step, _p(hist)))
    del keep, keep2
    return out, hist


def rel_linf(a: np.ndarray, b: np.ndarray) -> float:
    """tests/support/test_util.cpp:126-135: max|a-b| / max(max|b|, 1e-12)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b)) / max(float(np.max(np.abs(b))) if b.size else 0.0, 1e-12)) if a.size else 0.0


# ---- file-level I/O (graph_io.cpp:19-143, wav.cpp:39-133) -----------------------------------

def _text(fn, *args) -> str:
    n = _i64()
    _check(fn(*args, None, 0, ctypes.byref(n)))
    buf = ctypes.create_string_buffer(n.value + 1)
    _check(fn(*args, buf, n.value + 1, ctypes.byref(n)))
    return buf.raw[: n.value].decode()


def graph_to_json(types, edges, params: Optional[Dict[int, np.ndarray]] = None) -> str:
    types = np.ascontiguousarray(types, dtype=np.int32)
    edges = np.ascontiguousarray(edges, dtype=np.int32).reshape(-1, 4)
    ptrs, rows, _keep = _table_ptrs(params or {})
    return _text(lib().ref_graph_to_json, _p(types), len(types), _p(edges), len(edges), ptrs, _p(rows))


def _doc(h):
    try:
        nn, ne = _i32(), _i32()
        rows = np.zeros(10, dtype=np.int32)
        _check(lib().ref_doc_info(h, ctypes.byref(nn), ctypes.byref(ne), _p(rows)))
        t = np.zeros(nn.value, dtype=np.int32)
        e = np.zeros((ne.value, 4), dtype=np.int32)
        _check(lib().ref_doc_graph(h, _p(t), _p(e)))
        params = {}
        for ti in range(10):
            if rows[ti] >= 0:
                m = np.zeros((int(rows[ti]), WIDTHS[ti]))
                _check(lib().ref_doc_params(h, ti, _p(m)))
                params[ti] = m
        return t, e, params
    finally:
        lib().ref_doc_destroy(h)


def graph_from_json(text: str):
    """-> (types, edges[E][4], {type: table})"""
    h = _vp()
    _check(lib().ref_graph_from_json(text.encode(), ctypes.byref(h)))
    return _doc(h)


def load_graph(path: str):
    h = _vp()
    _check(lib().ref_load_graph(os.fsencode(path), ctypes.byref(h)))
    return _doc(h)


def save_graph(types, edges, params, path: str) -> None:
    types = np.ascontiguousarray(types, dtype=np.int32)
    edges = np.ascontiguousarray(edges, dtype=np.int32).reshape(-1, 4)
    ptrs, rows, _keep = _table_ptrs(params or {})
    _check(lib().ref_save_graph(_p(types), len(types), _p(edges), len(edges), ptrs, _p(rows), os.fsencode(path)))


def export_dot(types, edges) -> str:
    types = np.ascontiguousarray(types, dtype=np.int32)
    edges = np.ascontiguousarray(edges, dtype=np.int32).reshape(-1, 4)
    return _text(lib().ref_export_dot, _p(types), len(types), _p(edges), len(edges))


def write_wav(samples: np.ndarray, path: str, sample_rate: float = 44100.0) -> None:
    a = np.ascontiguousarray(samples, dtype=np.float64)
    if a.ndim == 2:
        a = a[None]
    _check(lib().ref_write_wav(_p(a), a.shape[0], a.shape[1], a.shape[2], float(sample_rate), os.fsencode(path)))


def read_wav(path: str):
    n, fs = _i64(), _dbl()
    _check(lib().ref_read_wav(os.fsencode(path), None, 0, ctypes.byref(n), ctypes.byref(fs)))
    out = np.zeros((1, 2, n.value))
    _check(lib().ref_read_wav(os.fsencode(path), _p(out), out.size, ctypes.byref(n), ctypes.byref(fs)))
    return out, fs.value
