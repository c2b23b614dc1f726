"""Graph-level sharding across GPUs (one process per GPU, no forward collective).

Graphs are independent (graph-level parallelism, `graph.cpp:116-128` disjoint_union), so a
batch of graphs is split across ranks and every rank renders its shard as ONE disjoint
union (one plan, one arena, one CUDA graph). Assignment is LPT (longest processing time
first) on a per-graph cost in node-samples weighted by processor type, so ranks finish
together; the assignment is a pure function of the inputs, identical on every rank.
"""
from __future__ import annotations

import heapq
from typing import List, Sequence, Tuple

import numpy as np

# Relative per-node-sample cost by NodeType (in, out, mix, gain, eq, comp, gate, imager,
# reverb, delay), from the measured per-step device times of config 2 (profiles/).
TYPE_WEIGHT = np.array([0.0, 0.5, 1.0, 1.0, 6.0, 3.0, 3.0, 1.0, 10.0, 10.0])


def graph_cost(node_types: Sequence[int], length: int, batch: int = 1) -> float:
    t = np.asarray(node_types, dtype=np.int64)
    return float(TYPE_WEIGHT[t].sum()) * length * batch


def lpt_shards(costs: Sequence[float], world: int) -> List[List[int]]:
    """Indices of the graphs each rank renders; ties broken by index (deterministic)."""
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    heap: List[Tuple[float, int]] = [(0.0, r) for r in range(world)]
    shards: List[List[int]] = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        shards[r].append(i)
        heapq.heappush(heap, (load + costs[i], r))
    return [sorted(s) for s in shards]


def union_arrays(graphs: Sequence[Tuple[np.ndarray, np.ndarray]]) -> Tuple[np.ndarray, np.ndarray]:
    """(types, edges) of the disjoint union, members in order (`graph.cpp:116-128`)."""
    types, edges, off = [], [], 0
    for t, e in graphs:
        types.append(np.asarray(t, dtype=np.int32))
        edges.append(np.asarray(e, dtype=np.int32).reshape(-1, 4) + np.array([off, off, 0, 0], dtype=np.int32))
        off += len(t)
    if not types:
        return np.zeros(0, dtype=np.int32), np.zeros((0, 4), dtype=np.int32)
    return np.concatenate(types), np.concatenate(edges)
