"""ORACLE — test infrastructure only (tests/, __graft_entry__.smoke(),
bench.py's cpu_baseline / --impl reference leg).  Never imported by the
product package.

numpy restatement of the reference policy rollout and its REINFORCE
gradient, structured like the reference (recomputes the SEL forward over the
candidate set at every step, re-gathers h_d over all placed vertices, builds
a reverse-mode tape) so it is an independent check of the CUDA path's
factorised per-vertex tables:

  _standardize            flowplace/policy.py:101-105
  GraphEncoding.build     flowplace/policy.py:120-146
  gnn_encode              flowplace/policy.py:149-173
  sel_forward             flowplace/policy.py:186-204
  plc_forward             flowplace/policy.py:207-223
  dynamic_device_features flowplace/policy.py:226-247 (+ timeline.py:30-58)
  _sample                 flowplace/policy.py:301-322
  rollout                 flowplace/policy.py:324-402
  tape ops / backward     flowplace/nn.py:62-224
  CriticalPathRule        flowplace/heuristics.py:65-91
  RL / imitation loss     flowplace/training.py:144, 200-216

Pinned against traces / encodings / gradients dumped from the reference
(tests/golden/policy_cases.json via tests/golden/make_golden.py).

Sampling: the reference draws from numpy PCG64, which no GPU reproduces; the
oracle instead takes the decision per step as (a) forced indices, (b) greedy,
(c) explicit uniforms (u1 for the epsilon test, u2 for the index) — the same
Philox4x32-10 uniforms the CUDA sampler consumes (``philox_uniforms``).
"""

from __future__ import annotations

import numpy as np

# ----------------------------------------------------------------------------
# reverse-mode tape (float64, rank-2), the op set of flowplace/nn.py
# ----------------------------------------------------------------------------


class T:
    __slots__ = ("v", "g", "ins", "back", "need")

    def __init__(self, v, ins=(), back=None, need=False):
        self.v = np.atleast_2d(np.asarray(v, dtype=np.float64))
        self.ins = ins
        self.back = back
        self.need = need or any(i.need for i in ins)
        self.g = None


def leaf(v, need=False):
    return T(v, need=need)


def _fit(g, shape):
    if g.shape == shape:
        return g
    if shape[0] == 1 and g.shape[0] != 1:
        g = g.sum(axis=0, keepdims=True)
    if shape[1] == 1 and g.shape[1] != 1:
        g = g.sum(axis=1, keepdims=True)
    return g


def mm(a, b):
    return T(a.v @ b.v, (a, b), lambda g: (g @ b.v.T, a.v.T @ g))


def add(a, b):
    return T(a.v + b.v, (a, b), lambda g: (_fit(g, a.v.shape), _fit(g, b.v.shape)))


def mul(a, b):
    return T(a.v * b.v, (a, b), lambda g: (_fit(g * b.v, a.v.shape), _fit(g * a.v, b.v.shape)))


def smul(a, c):
    return T(a.v * c, (a,), lambda g: (g * c,))


def sadd(a, c):
    return T(a.v + c, (a,), lambda g: (g,))


def cat(parts, axis=1):
    sizes = np.cumsum([p.v.shape[axis] for p in parts])[:-1]
    return T(np.concatenate([p.v for p in parts], axis=axis), tuple(parts),
             lambda g: tuple(np.split(g, sizes, axis=axis)))


def gather(a, idx):
    idx = np.asarray(idx, dtype=np.intp).reshape(-1)

    def back(g):
        out = np.zeros_like(a.v)
        np.add.at(out, idx, g)
        return (out,)

    return T(a.v[idx], (a,), back)


def rep(a, k):
    return T(np.repeat(a.v, k, axis=0), (a,), lambda g: (g.sum(axis=0, keepdims=True),))


def segsum(a, seg, m):
    seg = np.asarray(seg, dtype=np.intp).reshape(-1)
    out = np.zeros((m, a.v.shape[1]))
    np.add.at(out, seg, a.v)
    return T(out, (a,), lambda g: (g[seg],))


def leaky(a, s):
    pos = a.v > 0
    return T(np.where(pos, a.v, s * a.v), (a,), lambda g: (g * np.where(pos, 1.0, s),))


def softmax(a):
    e = np.exp(a.v - a.v.max(axis=1, keepdims=True))
    p = e / e.sum(axis=1, keepdims=True)
    return T(p, (a,), lambda g: (p * (g - (g * p).sum(axis=1, keepdims=True)),))


def log(a):
    return T(np.log(a.v), (a,), lambda g: (g / a.v,))


def total(a):
    return T([[a.v.sum()]], (a,), lambda g: (np.full_like(a.v, g.reshape(-1)[0]),))


def reshape(a, shape):
    return T(a.v.reshape(shape), (a,), lambda g: (g.reshape(a.v.shape),))


def backward(loss):
    order, seen, stack = [], set(), [(loss, False)]
    while stack:
        node, done = stack.pop()
        if done:
            order.append(node)
            continue
        if id(node) in seen or not node.need:
            continue
        seen.add(id(node))
        stack.append((node, True))
        stack.extend((p, False) for p in node.ins)
    grads = {id(loss): np.ones((1, 1))}
    for node in reversed(order):
        g = grads.pop(id(node), None)
        if g is None:
            continue
        node.g = g if node.g is None else node.g + g
        if node.back is None:
            continue
        for p, pg in zip(node.ins, node.back(g)):
            if p.need:
                grads[id(p)] = grads[id(p)] + pg if id(p) in grads else pg


# ----------------------------------------------------------------------------
# Philox4x32-10 uniforms (the CUDA sampler's stream, csrc/fp_common.cuh)
# ----------------------------------------------------------------------------

_M = np.uint64(0xFFFFFFFF)


def philox4x32_10(ctr, key):
    c = [np.uint64(int(x)) for x in ctr]
    k0, k1 = np.uint64(int(key[0])), np.uint64(int(key[1]))
    for r in range(10):
        if r:
            k0 = (k0 + np.uint64(0x9E3779B9)) & _M
            k1 = (k1 + np.uint64(0xBB67AE85)) & _M
        p0 = np.uint64(0xD2511F53) * c[0]
        p1 = np.uint64(0xCD9E8D57) * c[2]
        c = [((p1 >> np.uint64(32)) ^ c[1] ^ k0) & _M, p1 & _M,
             ((p0 >> np.uint64(32)) ^ c[3] ^ k1) & _M, p0 & _M]
    return [int(x) for x in c]


def philox_uniforms(seed: int, episode: int, step: int, head: int) -> tuple[float, float]:
    x = philox4x32_10((episode & 0xFFFFFFFF, step, head, 0),
                      (seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF))
    s = 2.0 ** -53
    u1 = (((x[1] << 32) | x[0]) >> 11) * s
    u2 = (((x[3] << 32) | x[2]) >> 11) * s
    return u1, u2


# ----------------------------------------------------------------------------
# policy
# ----------------------------------------------------------------------------


def standardize(mat):
    mean = mat.mean(axis=0) if mat.size else np.zeros(mat.shape[1])
    std = mat.std(axis=0) if mat.size else np.ones(mat.shape[1])
    std = np.where(std < 1e-12, 1.0, std)
    return (mat - mean) / std


class Ctx:
    """Per-graph constants (reference PolicyContext / GraphEncoding)."""

    def __init__(self, graph, cluster, hidden, k_rounds, slope=0.01, shared=False,
                 features=None):
        from paper_2505_23131_b200.features import static_features
        self.g, self.cl = graph, cluster
        self.h, self.K, self.slope, self.shared = hidden, k_rounds, slope, shared
        self.f = features if features is not None else static_features(graph, cluster.comm_factor)
        self.x = standardize(self.f.matrix)
        src, dst, cost = [], [], []
        for u, v in graph.edges:
            c = graph.vertices[u].output_bytes * self.f.comm_factor
            src += [u, v]
            dst += [v, u]
            cost += [c, c]
        ca = np.asarray(cost, dtype=np.float64).reshape(-1, 1)
        if ca.size:
            em, es = float(ca.mean()), float(ca.std()) or 1.0
        else:
            em, es = 0.0, 1.0
        es = es if es >= 1e-12 else 1.0
        self.src = np.asarray(src, dtype=np.intp)
        self.dst = np.asarray(dst, dtype=np.intp)
        self.edge = (ca - em) / es


def encode(P, ctx, head, dyn=None):
    pre = "enc" if ctx.shared else head
    n = len(ctx.g)
    H = leaf(np.concatenate([ctx.x, np.zeros((n, 2)) if dyn is None else dyn], axis=1))
    e = leaf(ctx.edge)
    for k in range(ctx.K):
        if ctx.src.size:
            m = cat([gather(H, ctx.src), gather(H, ctx.dst), e])
            m = leaky(add(mm(m, P[f"{pre}.gnn{k}.psi.w"]), P[f"{pre}.gnn{k}.psi.b"]), ctx.slope)
            agg = segsum(m, ctx.dst, n)
        else:
            agg = leaf(np.zeros((n, ctx.h)))
        H = leaky(add(mm(cat([H, agg]), P[f"{pre}.gnn{k}.phi.w"]), P[f"{pre}.gnn{k}.phi.b"]),
                  ctx.slope)
    return H


def _head(P, head, emb, slope):
    hid = leaky(add(mm(emb, P[f"{head}.head1.w"]), P[f"{head}.head1.b"]), slope)
    return add(mm(hid, P[f"{head}.head2.w"]), P[f"{head}.head2.b"])


def sel_probs(P, ctx, H, cands):
    bp = [ctx.f.b_paths[v] for v in cands]
    tp = [ctx.f.t_paths[v] for v in cands]
    hb = segsum(gather(H, np.concatenate(bp)),
                np.concatenate([[i] * len(p) for i, p in enumerate(bp)]), len(cands))
    ht = segsum(gather(H, np.concatenate(tp)),
                np.concatenate([[i] * len(p) for i, p in enumerate(tp)]), len(cands))
    z = add(mm(gather(leaf(ctx.x), cands), P["sel.z.w"]), P["sel.z.b"])
    s = _head(P, "sel", cat([gather(H, cands), hb, ht, z]), ctx.slope)
    return softmax(reshape(s, (1, len(cands))))


def plc_probs(P, ctx, H, v, placed, placed_dev, xdn):
    D = ctx.cl.device_count
    hv = rep(gather(H, [v]), D)
    hd = segsum(gather(H, placed), placed_dev, D) if placed else leaf(np.zeros((D, ctx.h)))
    y = add(mm(leaf(xdn), P["plc.y.w"]), P["plc.y.b"])
    z = rep(add(mm(gather(leaf(ctx.x), [v]), P["plc.z.w"]), P["plc.z.b"]), D)
    s = _head(P, "plc", cat([hv, hd, y, z]), ctx.slope)
    return softmax(reshape(s, (1, D)))


class Timeline:
    def __init__(self, g, cl):
        self.g, self.cl = g, cl
        self.avail = [0.0] * cl.device_count
        self.aflops = [0.0] * cl.device_count
        self.dev = [-1] * len(g)
        self.start = [0.0] * len(g)
        self.end = [0.0] * len(g)

    def arrival(self, p, d):
        if self.g.is_entry(p):
            return 0.0
        s = self.dev[p]
        if s < 0:
            raise ValueError(f"predecessor {p} is not assigned yet")
        tr = 0.0 if s == d else self.g.vertices[p].output_bytes * self.cl.comm_factor / \
            self.cl.bandwidth[s][d]
        return self.end[p] + tr

    def ready(self, v, d):
        return max((self.arrival(u, d) for u in self.g.preds(v)), default=0.0)

    def earliest(self, v, d):
        return max(self.avail[d], self.ready(v, d))

    def commit(self, v, d):
        self.dev[v] = d
        self.aflops[d] += self.g.vertices[v].flops
        if self.g.is_entry(v):
            return
        st = self.earliest(v, d)
        self.start[v] = st
        self.end[v] = st + self.g.vertices[v].flops / self.cl.rates[d]
        self.avail[d] = self.end[v]


def device_features(g, tl, v, D):
    out = np.zeros((D, 5))
    preds = g.preds(v)
    for p in preds:
        if tl.dev[p] < 0:
            raise ValueError(f"predecessor {p} of vertex {v} is unassigned")
    for d in range(D):
        out[d, 0] = tl.aflops[d]
        loc = [p for p in preds if tl.dev[p] == d]
        out[d, 1] = sum(g.vertices[p].flops for p in loc)
        out[d, 2] = min((tl.start[p] for p in loc), default=0.0)
        out[d, 3] = tl.ready(v, d)
        out[d, 4] = tl.earliest(v, d)
    return out


def sample(probs, eps, how):
    """how: ("forced", idx) | ("greedy",) | ("uniform", u1, u2)."""
    k = probs.v.shape[1]
    mix = sadd(smul(probs, 1.0 - eps), eps / k)
    p = probs.v[0]
    if how[0] == "forced":
        idx = int(how[1])
    elif how[0] == "greedy":
        idx = int(np.argmax(p))
    else:
        _, u1, u2 = how
        if u1 < eps:
            idx = min(int(u2 * k), k - 1)
        else:
            cum = np.cumsum(p)
            idx = min(int(np.searchsorted(cum, u2 * cum[-1], side="right")), k - 1)
    lm = log(sadd(mix, 1e-30))
    lp = gather(reshape(lm, (k, 1)), [idx])
    ent = smul(total(mul(mix, lm)), -1.0)
    return idx, lp, ent


def rollout(P, ctx, eps, mode="uniform", seed=0, episode=0, forced=None, teacher=False,
            greedy=False, per_step=False):
    """One episode.  mode: "uniform" (Philox draws), "forced" (``forced`` =
    [(v, d)] per step), "teacher" (CriticalPathRule) or "greedy".
    per_step: re-encode before every decision with the dynamic columns of the
    vertices placed so far (reference policy.py:353-371).
    Returns dict(assign, steps=[...], lps=[tape], ents=[tape])."""
    g, D = ctx.g, ctx.cl.device_count
    n = len(g)
    tl = Timeline(g, ctx.cl)
    cands = sorted(g.entry_vertices())
    left = [len(g.preds(v)) for v in range(n)]
    placed, placed_dev = [], []
    dyn = np.zeros((n, 2))
    if not per_step:
        Hs, Hp = encode(P, ctx, "sel"), encode(P, ctx, "plc")
    tlev = ctx.f.t_level
    steps, lps, ents = [], [], []
    for t in range(n):
        cand = tuple(cands)
        if per_step:
            Hs, Hp = encode(P, ctx, "sel", dyn), encode(P, ctx, "plc", dyn)
        ps = sel_probs(P, ctx, Hs, cands)
        if mode == "forced":
            fv = forced[t][0]
            if fv not in cands:
                raise ValueError(f"forced vertex {fv} outside candidates {cands}")
            how = ("forced", cands.index(fv))
        elif mode == "teacher":
            best = max(tlev[v] for v in cands)
            how = ("forced", cands.index([v for v in cands if tlev[v] == best][0]))
        elif mode == "greedy":
            how = ("greedy",)
        else:
            how = ("uniform",) + philox_uniforms(seed, episode, t, 0)
        i, lps_, ents_ = sample(ps, eps, how)
        v = cands[i]
        xd = device_features(g, tl, v, D)
        pp = plc_probs(P, ctx, Hp, v, placed, placed_dev, standardize(xd))
        if mode == "forced":
            how = ("forced", forced[t][1])
        elif mode == "teacher":
            best_d, best_t = 0, None
            for d in range(D):
                e = tl.earliest(v, d)
                if best_t is None or e < best_t:
                    best_d, best_t = d, e
            how = ("forced", best_d)
        elif mode == "greedy":
            how = ("greedy",)
        else:
            how = ("uniform",) + philox_uniforms(seed, episode, t, 1)
        j, lpp, entp = sample(pp, eps, how)
        tl.commit(v, j)
        dyn[v, 0] = 1.0
        dyn[v, 1] = (j + 1) / D
        placed.append(v)
        placed_dev.append(j)
        cands.remove(v)
        for w in g.succs(v):
            left[w] -= 1
            if left[w] == 0:
                cands.append(w)
        cands.sort()
        steps.append(dict(candidates=cand, vertex=v, device=j,
                          sel_logprob=float(lps_.v[0, 0]), plc_logprob=float(lpp.v[0, 0]),
                          sel_entropy=float(ents_.v[0, 0]), plc_entropy=float(entp.v[0, 0]),
                          sel_argmax=cand[int(np.argmax(ps.v[0]))],
                          plc_argmax=int(np.argmax(pp.v[0])), xd=xd,
                          sel_probs=ps.v[0].copy(), plc_probs=pp.v[0].copy()))
        lps += [lps_, lpp]
        ents += [ents_, entp]
    return dict(assign=list(tl.dev), steps=steps, lps=lps, ents=ents)


def leaves(params, need=True):
    return {k: leaf(getattr(v, "data", v), need=need) for k, v in params.items()}


def rl_gradients(params, ctx, eps, advantage, entropy_weight, **kw):
    """Gradient of loss = -(adv * sum lp + w * sum ent) for one episode
    (training.py:200-216); returns (grads by name, rollout record)."""
    P = leaves(params)
    ro = rollout(P, ctx, eps, **kw)
    obj = smul(total(cat(ro["lps"])), advantage)
    if entropy_weight > 0:
        obj = add(obj, smul(total(cat(ro["ents"])), entropy_weight))
    backward(smul(obj, -1.0))
    return {k: (t.g if t.g is not None else np.zeros_like(t.v)) for k, t in P.items()}, ro
