"""Synthetic workloads of the BASELINE configs (test and benchmark support, NOT the product).

The generators restate the reference's own bit-for-bit, so the GPU path and the reference CPU
renderer (oracle/_ref) see identical inputs:
  * generate_console — `proj/src/console.cpp:10-44` (libmgbwork.so, mt19937 order kept);
  * random_legal_params — `proj/tests/support/test_util.cpp:63-113` (fresh mt19937(seed));
  * generate_large_console — config 4's 966-node graph (SURVEY.md §8d recipe; the reference's
    generator tops out at 8K+6 nodes), no RNG.
The config builders below are the ONE definition of each BASELINE workload, shared by bench.py
and the full-size parity tests (tests/test_fullsize_gpu.py).
"""
from __future__ import annotations

import ctypes
import os
from typing import Dict, List, Sequence, Tuple

import numpy as np

import paper_2408_03204_b200 as mg
from paper_2408_03204_b200 import NodeType, NUM_NODE_TYPES, param_width

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = ctypes.CDLL(os.path.join(_HERE, "libmgbwork.so"))
_vp, _i32, _u32, _dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint32, ctypes.c_double
_lib.wl_last_error.restype = ctypes.c_char_p
_lib.wl_generate_console.restype = _i32
_lib.wl_generate_console.argtypes = [_i32, _dbl, _u32, _vp, _i32, _vp, _i32, ctypes.POINTER(_i32), ctypes.POINTER(_i32)]
_lib.wl_random_legal_params.restype = _i32
_lib.wl_random_legal_params.argtypes = [_vp, _i32, _u32, _vp]

FS = 44100.0
L2 = 1 << 17          # configs 2, 3, 5: stereo 2^17 samples
L4 = 441000           # config 4: 10 s
PRUNE = 0.3


def _check(st: int) -> None:
    if st != 0:
        raise ValueError(_lib.wl_last_error().decode())


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def generate_console_arrays(tracks: int, prune: float = 0.0, seed: int = 0) -> Tuple[np.ndarray, np.ndarray]:
    """`console.cpp:10-44` as (types [V], edges [E, 4]) int32 arrays."""
    cap_n, cap_e = 8 * tracks + 16, 10 * tracks + 16
    t = np.zeros(cap_n, dtype=np.int32)
    e = np.zeros((cap_e, 4), dtype=np.int32)
    nn, ne = _i32(), _i32()
    _check(_lib.wl_generate_console(tracks, prune, seed, _ptr(t), cap_n, _ptr(e), cap_e, ctypes.byref(nn), ctypes.byref(ne)))
    return t[:nn.value].copy(), e[:ne.value].copy()


def generate_console(tracks: int, prune: float = 0.0, seed: int = 0) -> "mg.Graph":
    """`console.cpp:10-44`."""
    return mg.Graph.from_arrays(*generate_console_arrays(tracks, prune, seed))


def random_legal_params(node_types: Sequence[int], seed: int) -> Dict[NodeType, np.ndarray]:
    """`tests/support/test_util.cpp:63-113` with a fresh mt19937(seed), original row order."""
    counts: Dict[int, int] = {}
    for t in node_types:
        if param_width(t) > 0:
            counts[int(t)] = counts.get(int(t), 0) + 1
    out = {NodeType(t): np.zeros((n, param_width(t))) for t, n in sorted(counts.items())}
    tt = np.ascontiguousarray(np.asarray([int(x) for x in node_types], dtype=np.int32))
    ptrs = (_vp * NUM_NODE_TYPES)()
    for t, m in out.items():
        ptrs[int(t)] = m.ctypes.data
    _check(_lib.wl_random_legal_params(_ptr(tt), len(tt), seed, ptrs))
    return out


def generate_large_console_arrays(tracks: int = 64) -> Tuple[np.ndarray, np.ndarray]:
    """BASELINE config 4's pruning-scale graph: per track in -> e c n s g e c n s g (a doubled
    channel strip), whose last gain feeds the mix bus directly and through two sends (delay ->
    gain, reverb -> gain); bus mix -> e c s g -> out. 15 nodes and 17 edges per track (64
    tracks: 966 nodes, 1093 edges). Insertion order follows console.cpp (per-track nodes, then
    the bus). Synthetic: no RNG, parameters come from random_legal_params."""
    if tracks < 1:
        raise ValueError("generate_large_console: need at least one track")
    T = NodeType
    types: List[int] = []
    edges: List[Tuple[int, int]] = []
    sends: List[int] = []

    def node(t):
        types.append(int(t))
        return len(types) - 1

    def chain(ts):
        ids = [node(t) for t in ts]
        for a, b in zip(ids, ids[1:]):
            edges.append((a, b))
        return ids[0], ids[-1]

    strip = [T.EQ, T.COMPRESSOR, T.NOISEGATE, T.IMAGER, T.GAIN] * 2
    for _ in range(tracks):
        i = node(T.IN)
        first, last = chain(strip)
        edges.append((i, first))
        for fx in (T.DELAY, T.REVERB):
            s0, s1 = chain([fx, T.GAIN])
            edges.append((last, s0))
            sends.append(s1)
        sends.append(last)
    bus = node(T.MIX)
    for s in sends:
        edges.append((s, bus))
    b0, b1 = chain([T.EQ, T.COMPRESSOR, T.IMAGER, T.GAIN])
    edges.append((bus, b0))
    out = node(T.OUT)
    edges.append((b1, out))
    e = np.zeros((len(edges), 4), dtype=np.int32)
    e[:, :2] = np.asarray(edges, dtype=np.int32)
    return np.asarray(types, dtype=np.int32), e


def sources(n: int, length: int, batch: int = 1, base_seed: int = 1000) -> np.ndarray:
    """[n][batch][2][length] fp64: uniform_noise(2 L, base_seed + k) per source (`bench.cpp:33-40`)."""
    return np.stack([np.stack([mg.uniform_noise(2 * length, base_seed + k + 100 * b).reshape(2, length)
                               for b in range(batch)]) for k in range(n)])


# ---- BASELINE configs ---------------------------------------------------------------------------

def config2():
    """Config 2: generate_console(16, p=0.3, seed=16) — the reference bench's K=16 graph (121
    nodes, 139 edges) — stereo 2^17, params random_legal_params(seed 2024)."""
    t, e = generate_console_arrays(16, PRUNE, 16)
    return t, e, random_legal_params(t, 2024)


def config3_members(step: int, graphs: int = 64) -> List[Tuple[np.ndarray, np.ndarray]]:
    """Config 3, batch `step`: 64 consoles, K_i uniform in [4, 32] (numpy default_rng(step)),
    p = 0.3, seed 1000*step + i — topology re-drawn every step."""
    rng = np.random.default_rng(step)
    return [generate_console_arrays(int(rng.integers(4, 33)), PRUNE, 1000 * step + i) for i in range(graphs)]


def config3_params_seed(step: int) -> int:
    return 5000 + step


def config5_graphs(n: int = 512, seed: int = 5) -> List[Tuple[np.ndarray, np.ndarray]]:
    """Config 5: 512 consoles built as config 3's (K_i in [4, 32], p = 0.3), fixed topology."""
    rng = np.random.default_rng(seed)
    return [generate_console_arrays(int(rng.integers(4, 33)), PRUNE, 50000 + i) for i in range(n)]


def config5_member_params(i: int, t: np.ndarray) -> Dict[NodeType, np.ndarray]:
    """Parameters of config-5 graph i (original row order; seeded per graph, so a graph's
    parameters do not depend on which shard or union it is rendered in)."""
    return random_legal_params(t, 70000 + i)


def union_params(members_t: Sequence[np.ndarray], per_member: Sequence[Dict[NodeType, np.ndarray]]):
    """concat_params (`graph.cpp:171-186`): member tables stacked in member order."""
    out: Dict[NodeType, List[np.ndarray]] = {}
    for p in per_member:
        for ty, tab in p.items():
            out.setdefault(NodeType(int(ty)), []).append(np.asarray(tab))
    return {ty: np.concatenate(v) for ty, v in out.items()}


def source_bank(rows: int = 64, length: int = L2) -> np.ndarray:
    """[rows][1][2][length] fp64 noise bank; input k of a union plan takes row k % rows."""
    return sources(rows, length)
