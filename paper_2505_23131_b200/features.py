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
    matrix: np.ndarray
    b_paths: tuple[tuple[int, ...], ...]
    t_paths: tuple[tuple[int, ...], ...]
    comm_factor: float

    @property
    def t_level(self) -> np.ndarray:
        return self.matrix[:, T_LEVEL]

    @property
    def b_level(self) -> np.ndarray:
        return self.matrix[:, B_LEVEL]


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


def static_features(graph: DataflowGraph,
                    comm_factor: float = DEFAULT_COMM_FACTOR) -> StaticGraphFeatures:
    n = len(graph)
    order = topo_order(graph)
    mat = np.zeros((n, 5), dtype=np.float64)
    cc = [graph.vertices[u].output_bytes * comm_factor for u in range(n)]
    for v in range(n):
        mat[v, COMPUTE_COST] = graph.vertices[v].flops
        mat[v, IN_COMM_SUM] = sum(cc[u] for u in graph.preds(v))
        mat[v, OUT_COMM_SUM] = cc[v] * len(graph.succs(v))
    t_next = _longest(graph, reversed(order), graph.succs, lambda v, w: cc[v], mat, T_LEVEL)
    b_next = _longest(graph, order, graph.preds, lambda v, u: cc[u], mat, B_LEVEL)
    return StaticGraphFeatures(mat, tuple(_walk(v, b_next) for v in range(n)),
                               tuple(_walk(v, t_next) for v in range(n)), comm_factor)
