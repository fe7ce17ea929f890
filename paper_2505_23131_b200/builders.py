"""Synthetic workload graphs for the hot path (fixtures, not product logic).

* ``build_chainmm`` / ``build_ffnn`` reproduce the reference builders
  (``builders.py:243-281``) vertex for vertex — same ids, labels, edges and
  meta-ops — so bench configs 1/2 run on the reference's exact graphs
  (checked against golden JSON dumped from the reference).
* ``build_llama_block`` / ``build_llama_layer`` are NEW (the reference has no
  Llama builder): a Llama-7B decoder block composed from the
  same blocked primitives (RMSNorm, Q/K/V, RoPE, K^T, QK^T, scale, row
  softmax, PV, O, residual, SwiGLU FFN, residual) at shard_grid=2; the layer
  adds the final RMSNorm, LM head and vocabulary softmax.
* ``sparse_dag`` is the seeded sparse generator of SURVEY §8(d) config 5
  (the reference's ``random_dag`` is dense O(n^2), ``tests/util.py:77-97``).
"""

from __future__ import annotations

import numpy as np

from .graph import DataflowGraph, MetaOp, OpKind, Vertex

DTYPE_BYTES = 4


class BlockedGraph:
    """Accumulates a blocked tensor program as a dataflow graph.  A blocked
    matrix is a dict ``(i, j) -> vertex id`` over a g x g grid."""

    def __init__(self, g: int):
        if g < 1:
            raise ValueError(f"shard_grid must be >= 1, got {g}")
        self.g = g
        self.V: list[Vertex] = []
        self.E: list[tuple[int, int]] = []
        self.M: list[MetaOp] = []

    # -- plumbing ------------------------------------------------------------
    def _add(self, kind, flops, nbytes, label, srcs=()):
        vid = len(self.V)
        self.V.append(Vertex(vid, kind, int(flops), int(nbytes), label))
        self.E.extend((s, vid) for s in srcs)
        return vid

    def _group(self, shard, reduce=()):
        self.M.append(MetaOp(len(self.M), tuple(shard), tuple(reduce)))

    def _div(self, dim, what):
        if dim % self.g:
            raise ValueError(f"{what}={dim} is not divisible by shard_grid={self.g}")
        return dim // self.g

    def _cells(self):
        return [(i, j) for i in range(self.g) for j in range(self.g)]

    # -- inputs --------------------------------------------------------------
    def matrix(self, name, rows, cols):
        blk = self._div(rows, "rows") * self._div(cols, "cols") * DTYPE_BYTES
        return {c: self._add(OpKind.INPUT, 0, blk, f"{name}[{c[0]},{c[1]}]") for c in self._cells()}

    def vector(self, name, size):
        blk = self._div(size, "size") * DTYPE_BYTES
        return {j: self._add(OpKind.INPUT, 0, blk, f"{name}[{j}]") for j in range(self.g)}

    # -- blocked ops -----------------------------------------------------------
    def matmul(self, name, a, a_dims, b, b_dims):
        if a_dims[1] != b_dims[0]:
            raise ValueError(f"non-conformable dims: {a_dims} x {b_dims}")
        g = self.g
        br, bk = a_dims[0] // g, a_dims[1] // g
        bc = self._div(b_dims[1], "cols")
        self._div(a_dims[0], "rows")
        self._div(a_dims[1], "inner")
        out_b = br * bc * DTYPE_BYTES
        parts = {}
        for i, j in self._cells():
            parts[(i, j)] = [self._add(OpKind.MATMUL, 2 * br * bk * bc, out_b,
                                       f"{name}.p[{i},{j},{k}]", (a[(i, k)], b[(k, j)]))
                             for k in range(g)]
        adds, out = [], {}
        for c in self._cells():
            acc = parts[c][0]
            for step, p in enumerate(parts[c][1:]):
                acc = self._add(OpKind.ADD, br * bc, out_b, f"{name}.s[{c[0]},{c[1]}]#{step}",
                                (acc, p))
                adds.append(acc)
            out[c] = acc
        self._group([p for c in self._cells() for p in parts[c]], adds)
        return out, (a_dims[0], b_dims[1])

    def pointwise(self, name, kind, dims, *operands):
        """One vertex per block; each operand is a grid, a row-vector
        ``{j: id}`` (broadcast over rows, tagged ('col', vec)) or a
        column-vector ``{i: id}`` (tagged ('row', vec))."""
        br, bc = dims[0] // self.g, dims[1] // self.g
        out = {}
        for i, j in self._cells():
            srcs = []
            for op in operands:
                if isinstance(op, tuple):
                    tag, vec = op
                    srcs.append(vec[j] if tag == "col" else vec[i])
                else:
                    srcs.append(op[(i, j)])
            out[(i, j)] = self._add(kind, br * bc, br * bc * DTYPE_BYTES,
                                    f"{name}[{i},{j}]", srcs)
        self._group([out[c] for c in self._cells()])
        return out

    def row_reduce(self, name, a, dims, label):
        """Reduce each row-block across its g column blocks -> {i: id}."""
        br, bc = dims[0] // self.g, dims[1] // self.g
        red = {i: self._add(OpKind.REDUCTION, self.g * br * bc, br * DTYPE_BYTES,
                            f"{name}.{label}[{i}]", [a[(i, j)] for j in range(self.g)])
               for i in range(self.g)}
        self._group([red[i] for i in range(self.g)])
        return red

    def softmax_rows(self, name, a, dims):
        g = self.g
        br, bc = dims[0] // g, dims[1] // g
        mx = self.row_reduce(name, a, dims, "max")
        ex = {}
        for i, j in self._cells():
            ex[(i, j)] = self._add(OpKind.ELEMWISE, br * bc, br * bc * DTYPE_BYTES,
                                   f"{name}.exp[{i},{j}]", (a[(i, j)], mx[i]))
        self._group([ex[c] for c in self._cells()])
        sm = self.row_reduce(name, ex, dims, "sum")
        out = {}
        for i, j in self._cells():
            out[(i, j)] = self._add(OpKind.ELEMWISE, br * bc, br * bc * DTYPE_BYTES,
                                    f"{name}.div[{i},{j}]", (ex[(i, j)], sm[i]))
        self._group([out[c] for c in self._cells()])
        return out

    def transpose(self, name, a, dims):
        """K^T as a formation op: block (i, j) of the result reads a[(j, i)]."""
        br, bc = dims[1] // self.g, dims[0] // self.g
        out = {(i, j): self._add(OpKind.FORMATION, br * bc, br * bc * DTYPE_BYTES,
                                 f"{name}[{i},{j}]", (a[(j, i)],)) for i, j in self._cells()}
        self._group([out[c] for c in self._cells()])
        return out

    def rmsnorm(self, name, x, gain, dims):
        sq = self.pointwise(f"{name}.sq", OpKind.ELEMWISE, dims, x)
        ss = self.row_reduce(name, sq, dims, "ss")
        return self.pointwise(f"{name}.scale", OpKind.ELEMWISE, dims, x, ("row", ss),
                              ("col", gain))

    def finish(self) -> DataflowGraph:
        return DataflowGraph(tuple(self.V), tuple(self.E), tuple(self.M))


def build_chainmm(n: int, shard_grid: int) -> DataflowGraph:
    """(A x B) + (C x (D x E)), all n x n (reference ``builders.py:243-258``)."""
    if n < shard_grid:
        raise ValueError(f"matrix dim {n} smaller than shard_grid {shard_grid}")
    b = BlockedGraph(shard_grid)
    dims = (n, n)
    A, B, C, D, E = (b.matrix(x, n, n) for x in "ABCDE")
    ab, _ = b.matmul("AB", A, dims, B, dims)
    de, _ = b.matmul("DE", D, dims, E, dims)
    cde, _ = b.matmul("CDE", C, dims, de, dims)
    b.pointwise("OUT", OpKind.ADD, dims, ab, cde)
    return b.finish()


def build_ffnn(batch: int, d_in: int, d_hidden: int, d_out: int,
               shard_grid: int) -> DataflowGraph:
    """Softmax(ReLU(X W1 + b1) W2 + b2) (reference ``builders.py:261-281``)."""
    for name, dim in (("batch", batch), ("d_in", d_in), ("d_hidden", d_hidden),
                      ("d_out", d_out)):
        if dim < 1:
            raise ValueError(f"{name} must be positive, got {dim}")
    b = BlockedGraph(shard_grid)
    x = b.matrix("X", batch, d_in)
    w1 = b.matrix("W1", d_in, d_hidden)
    b1 = b.vector("b1", d_hidden)
    w2 = b.matrix("W2", d_hidden, d_out)
    b2 = b.vector("b2", d_out)
    h0, hd = b.matmul("mm1", x, (batch, d_in), w1, (d_in, d_hidden))
    h1 = b.pointwise("badd1", OpKind.ELEMWISE, hd, h0, ("col", b1))
    h2 = b.pointwise("relu", OpKind.ELEMWISE, hd, h1)
    y0, yd = b.matmul("mm2", h2, hd, w2, (d_hidden, d_out))
    y1 = b.pointwise("badd2", OpKind.ELEMWISE, yd, y0, ("col", b2))
    b.softmax_rows("smax", y1, yd)
    return b.finish()


def _llama(seq: int, emb: int, ffn: int, vocab: int | None, g: int) -> DataflowGraph:
    b = BlockedGraph(g)
    xd, wd, fd = (seq, emb), (emb, emb), (emb, ffn)
    X = b.matrix("X", *xd)
    Wq, Wk, Wv, Wo = (b.matrix(w, *wd) for w in ("Wq", "Wk", "Wv", "Wo"))
    W1, W3 = b.matrix("W1", *fd), b.matrix("W3", *fd)
    W2 = b.matrix("W2", ffn, emb)
    g1, g2 = b.vector("g_attn", emb), b.vector("g_ffn", emb)
    if vocab is not None:
        gf = b.vector("g_final", emb)
        Wlm = b.matrix("W_lm", emb, vocab)
    xn = b.rmsnorm("norm1", X, g1, xd)
    q, _ = b.matmul("Q", xn, xd, Wq, wd)
    k, _ = b.matmul("K", xn, xd, Wk, wd)
    v, _ = b.matmul("V", xn, xd, Wv, wd)
    q = b.pointwise("rope_q", OpKind.ELEMWISE, xd, q)
    k = b.pointwise("rope_k", OpKind.ELEMWISE, xd, k)
    kt = b.transpose("Kt", k, xd)
    s, sd = b.matmul("QKt", q, xd, kt, (emb, seq))
    s = b.pointwise("scale", OpKind.ELEMWISE, sd, s)
    p = b.softmax_rows("attn", s, sd)
    o, _ = b.matmul("PV", p, sd, v, xd)
    o, _ = b.matmul("O", o, xd, Wo, wd)
    h = b.pointwise("resid1", OpKind.ADD, xd, X, o)
    hn = b.rmsnorm("norm2", h, g2, xd)
    a1, ad = b.matmul("W1x", hn, xd, W1, fd)
    a3, _ = b.matmul("W3x", hn, xd, W3, fd)
    a1 = b.pointwise("silu", OpKind.ELEMWISE, ad, a1)
    gt = b.pointwise("gate", OpKind.ELEMWISE, ad, a1, a3)
    f, _ = b.matmul("W2x", gt, ad, W2, (ffn, emb))
    out = b.pointwise("resid2", OpKind.ADD, xd, h, f)
    if vocab is not None:
        on = b.rmsnorm("norm_f", out, gf, xd)
        lg, ld = b.matmul("LM", on, xd, Wlm, (emb, vocab))
        b.softmax_rows("vocab", lg, ld)
    return b.finish()


def build_llama_block(seq: int = 4096, emb: int = 4096, ffn: int = 11008,
                      shard_grid: int = 2) -> DataflowGraph:
    """Llama-7B decoder block (PAPER.md:596-606 dims), blocked at shard_grid."""
    return _llama(seq, emb, ffn, None, shard_grid)


def build_llama_layer(seq: int = 4096, emb: int = 4096, ffn: int = 11008,
                      vocab: int = 32000, shard_grid: int = 2) -> DataflowGraph:
    """Block + final RMSNorm + LM head + vocabulary softmax (largest graph)."""
    return _llama(seq, emb, ffn, vocab, shard_grid)


def sparse_dag(n: int, seed: int = 0, window: int = 64) -> DataflowGraph:
    """Seeded sparse DAG: the first max(1, n//20) vertices are inputs; every
    other vertex draws 1-3 distinct predecessors from the previous ``window``
    ids; flops U[2^20, 2^30), output bytes U[2^16, 2^22)."""
    rng = np.random.default_rng(seed)
    n_in = max(1, n // 20)
    verts, edges = [], []
    for v in range(n):
        nbytes = int(rng.integers(1 << 16, 1 << 22))
        if v < n_in:
            verts.append(Vertex(v, OpKind.INPUT, 0, nbytes, f"in{v}"))
            continue
        lo = max(0, v - window)
        k = min(int(rng.integers(1, 4)), v - lo)
        for u in sorted(rng.choice(np.arange(lo, v), size=k, replace=False).tolist()):
            edges.append((int(u), v))
        verts.append(Vertex(v, OpKind.OTHER, int(rng.integers(1 << 20, 1 << 30)), nbytes, f"op{v}"))
    return DataflowGraph(tuple(verts), tuple(edges))


def relabel(graph: DataflowGraph, seed: int = 0) -> DataflowGraph:
    """The same DAG under a random permutation of vertex ids -- destroys the
    id locality of ``sparse_dag`` (predecessors within a 64-id window), so
    per-message gathers of neighbour rows become random HBM accesses."""
    import dataclasses

    n = len(graph)
    perm = np.random.default_rng(seed).permutation(n)
    verts = [None] * n
    for v, x in enumerate(graph.vertices):
        verts[int(perm[v])] = dataclasses.replace(x, id=int(perm[v]))
    edges = tuple((int(perm[a]), int(perm[b])) for a, b in graph.edges)
    return DataflowGraph(tuple(verts), edges)
