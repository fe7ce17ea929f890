"""Static per-vertex features (host mirror of reference ``features.py:51-96``).

Columns of the n x 5 float64 matrix: compute cost, summed incoming comm
cost, outgoing comm cost x out-degree, t-level (longest path toward exits),
b-level (longest path toward entries).  Both levels include the vertex's own
cost; ties between equal-cost continuations keep the smallest neighbour id.
The per-vertex argmax paths feed the SEL path-sum embeddings and the levels
order the simulator's depth_first / breadth_first strategies, so the
arithmetic here follows the reference operation for operation.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .graph import DataflowGraph, topo_order

DEFAULT_COMM_FACTOR = 4.0
COMPUTE_COST, IN_COMM_SUM, OUT_COMM_SUM, T_LEVEL, B_LEVEL = range(5)


@dataclass
class StaticGraphFeatures:
    """``b_next[v]`` / ``t_next[v]`` are the argmax neighbours of the two
    longest-path sweeps (-1 at a path's end): the paths form two forests, and
    ``b_paths[v]`` = (v, b_next[v], b_next[b_next[v]], ...).  The explicit
    path tuples (reference ``features.py:88-95``) are materialised on first
    use only -- their total length grows like n * depth (2.7e8 entries at
    100k ops), so large graphs are handed to the GPU as the next arrays."""

    matrix: np.ndarray
    b_next: np.ndarray
    t_next: np.ndarray
    comm_factor: float

    @property
    def t_level(self) -> np.ndarray:
        return self.matrix[:, T_LEVEL]

    @property
    def b_level(self) -> np.ndarray:
        return self.matrix[:, B_LEVEL]

    @property
    def b_paths(self) -> tuple[tuple[int, ...], ...]:
        if getattr(self, "_b_paths", None) is None:
            nxt = self.b_next.tolist()
            self._b_paths = tuple(_walk(v, nxt) for v in range(len(nxt)))
        return self._b_paths

    @property
    def t_paths(self) -> tuple[tuple[int, ...], ...]:
        if getattr(self, "_t_paths", None) is None:
            nxt = self.t_next.tolist()
            self._t_paths = tuple(_walk(v, nxt) for v in range(len(nxt)))
        return self._t_paths

    def path_lengths(self, which: str) -> np.ndarray:
        """Length of every b- or t-path, from the next forest by pointer
        jumping (vectorised, O(n log depth))."""
        nxt = np.asarray(self.b_next if which == "b" else self.t_next, dtype=np.int64)
        length = np.ones(len(nxt), dtype=np.int64)
        ptr = nxt.copy()
        while (ptr >= 0).any():
            live = ptr >= 0
            tgt = np.where(live, ptr, 0)
            length = length + np.where(live, length[tgt], 0)
            ptr = np.where(live, ptr[tgt], -1)
        return length


def edge_comm_cost(graph: DataflowGraph, u: int, comm_factor: float) -> float:
    return graph.vertices[u].output_bytes * comm_factor


def _longest(graph, order, nbrs, cost_src, mat, col):
    """One longest-path sweep; ``cost_src(v, w)`` names whose output bytes
    the step between v and neighbour w carries."""
    nxt = [-1] * len(graph)
    for v in order:
        best, arg = 0.0, -1
        for w in nbrs(v):
            cand = cost_src(v, w) + mat[w, col]
            if arg == -1 or cand > best:
                best, arg = cand, w
        mat[v, col] = graph.vertices[v].flops + best
        nxt[v] = arg
    return nxt


def _walk(start: int, nxt: list[int]) -> tuple[int, ...]:
    out = [start]
    while nxt[out[-1]] != -1:
        out.append(nxt[out[-1]])
    return tuple(out)


# graphs from this size on use the native sweep (fp_static_features: the same
# arithmetic in C++, bit-identical; the Python loops take seconds at 100k+ ops)
NATIVE_MIN_N = 4096


def static_features(graph: DataflowGraph, comm_factor: float = DEFAULT_COMM_FACTOR,
                    native: bool | None = None) -> StaticGraphFeatures:
    n = len(graph)
    use_native = n >= NATIVE_MIN_N if native is None else native
    if use_native:
        return _static_features_native(graph, comm_factor)
    order = topo_order(graph)
    mat = np.zeros((n, 5), dtype=np.float64)
    cc = [graph.vertices[u].output_bytes * comm_factor for u in range(n)]
    for v in range(n):
        mat[v, COMPUTE_COST] = graph.vertices[v].flops
        mat[v, IN_COMM_SUM] = sum(cc[u] for u in graph.preds(v))
        mat[v, OUT_COMM_SUM] = cc[v] * len(graph.succs(v))
    t_next = _longest(graph, reversed(order), graph.succs, lambda v, w: cc[v], mat, T_LEVEL)
    b_next = _longest(graph, order, graph.preds, lambda v, u: cc[u], mat, B_LEVEL)
    return StaticGraphFeatures(mat, np.asarray(b_next, dtype=np.int32),
                               np.asarray(t_next, dtype=np.int32), comm_factor)


def _static_features_native(graph: DataflowGraph, comm_factor: float) -> StaticGraphFeatures:
    import ctypes

    from . import _native as N

    n = len(graph)
    c = graph.csr()
    mat = np.zeros((n, 5), dtype=np.float64)
    b_next = np.empty(n, dtype=np.int32)
    t_next = np.empty(n, dtype=np.int32)
    N.check(N.lib().fp_static_features(
        ctypes.c_int32(n), *[N.ptr(c[k]) for k in ("pred_indptr", "pred_indices", "succ_indptr",
                                                   "succ_indices", "flops", "obytes")],
        ctypes.c_double(comm_factor), N.ptr(mat), N.ptr(b_next), N.ptr(t_next)))
    return StaticGraphFeatures(mat, b_next, t_next, comm_factor)
