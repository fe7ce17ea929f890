"""Shared test fixtures (graphs/clusters) restated from the reference's
tests/util.py:18-97 so GPU-box tests need no reference checkout."""
from __future__ import annotations

import numpy as np

from paper_2505_23131_b200.cluster import ClusterSpec
from paper_2505_23131_b200.graph import DataflowGraph, MetaOp, OpKind, Vertex


def graph_from_golden(gd: dict) -> DataflowGraph:
    """Build without validation (golden cases include a deliberate cycle)."""
    vs = tuple(Vertex(v["id"], OpKind(v["op_kind"]), v["flops"], v["output_bytes"], v["label"])
               for v in gd["vertices"])
    ms = tuple(MetaOp(m["id"], tuple(m["shard_ops"]), tuple(m["reduce_ops"]))
               for m in gd.get("meta_ops", []))
    return DataflowGraph(vs, tuple(tuple(e) for e in gd["edges"]), ms)


def chain_graph(flops=(1000, 1000, 1000), bytes_=64) -> DataflowGraph:
    vs = [Vertex(0, OpKind.INPUT, 0, bytes_, "x")]
    es = []
    for i, f in enumerate(flops, start=1):
        vs.append(Vertex(i, OpKind.OTHER, f, bytes_, f"op{i}"))
        es.append((i - 1, i))
    return DataflowGraph(tuple(vs), tuple(es))


def fixture6() -> DataflowGraph:
    return DataflowGraph(
        (Vertex(0, OpKind.INPUT, 0, 64, "x"), Vertex(1, OpKind.MATMUL, 4000, 64, "m1"),
         Vertex(2, OpKind.MATMUL, 4000, 64, "m2"), Vertex(3, OpKind.OTHER, 1000, 64, "p1"),
         Vertex(4, OpKind.OTHER, 1000, 64, "p2"), Vertex(5, OpKind.REDUCTION, 500, 64, "r")),
        ((0, 1), (0, 2), (1, 3), (2, 4), (3, 5), (4, 5)))


def cluster2(rate=1000.0, bandwidth=256.0, **kw) -> ClusterSpec:
    return ClusterSpec.uniform(2, rate=rate, bandwidth=bandwidth, **kw)


def random_dag(rng: np.random.Generator, max_vertices: int = 8, edge_prob: float = 0.45):
    n = int(rng.integers(2, max_vertices + 1))
    edges, has_pred = [], [False] * n
    for u in range(n):
        for v in range(u + 1, n):
            if rng.random() < edge_prob:
                edges.append((u, v))
                has_pred[v] = True
    vs = []
    for v in range(n):
        if has_pred[v]:
            vs.append(Vertex(v, OpKind.OTHER, int(rng.integers(100, 5000)),
                             int(rng.integers(16, 256)), f"v{v}"))
        else:
            vs.append(Vertex(v, OpKind.INPUT, 0, int(rng.integers(16, 256)), f"v{v}"))
    return DataflowGraph(tuple(vs), tuple(edges))
