"""Stage I/II training on the GPU — mirror of reference ``flowplace/training.py``.

Reference semantics (``training.py:181-216``): per episode, reward = -makespan,
advantage = reward - mean(all previous returns), loss = -(adv * sum lp +
w * sum entropy), one SGD step with a linear lr schedule; epsilon linear
0.2 -> 0.  The B200 trainer runs B episodes per update (B per GPU, episodes
sharded over ranks):

    encode -> rollout+sim (REINFORCE rows) -> alpha_e = (mk_e + baseline)/B_g
    -> fp_pg_reduce -> fp_policy_backward -> NCCL allreduce([grad | sum r])
    -> SGD (lr at the batch's first episode index) -> baseline update

At B_global = 1 this is exactly the reference's per-episode update (the
baseline is the mean of all previous returns, kept globally across ranks).
"""

from __future__ import annotations

import ctypes
import itertools
import json
import math
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _native as N
from .cluster import ClusterSpec
from .graph import DataflowGraph
from .heuristics import Assignment, CriticalPathRule  # noqa: F401
from .params import (Params, init_policy_params, load_params, param_shapes, save_params)
from .policy import PolicyConfig, PolicyContext, is_native_teacher, teacher_actions
from .simulate import exec_time_batch

STAGES = ("imitation", "sim_rl", "system_rl")


@dataclass
class TrainConfig:
    episodes: int = 500
    lr0: float = 1e-4
    lr1: float = 1e-7
    epsilon0: float = 0.2
    entropy_weight: float = 1e-2
    seed: int = 0
    strategy: str = "fifo"

    def __post_init__(self):
        if self.episodes < 1:
            raise ValueError("episodes must be >= 1")
        if self.entropy_weight < 0:
            raise ValueError("entropy_weight must be >= 0")

    def to_dict(self) -> dict:
        return {"episodes": self.episodes, "lr0": self.lr0, "lr1": self.lr1,
                "epsilon0": self.epsilon0, "entropy_weight": self.entropy_weight,
                "seed": self.seed, "strategy": self.strategy}

    @classmethod
    def from_dict(cls, doc: dict) -> "TrainConfig":
        keys = ("episodes", "lr0", "lr1", "epsilon0", "entropy_weight", "seed", "strategy")
        return cls(**{k: doc[k] for k in keys if k in doc})


@dataclass
class LinearSchedule:
    """v0 at step 0, v1 at step ``total``, linear between (nn.py:244-256)."""

    v0: float
    v1: float
    total: int

    def value(self, step: int) -> float:
        if self.total <= 0:
            return self.v1
        frac = min(max(step, 0), self.total) / self.total
        return self.v0 * (1.0 - frac) + self.v1 * frac


class RewardTracker:
    """Baseline = mean of all previously observed returns (training.py:65-78)."""

    def __init__(self):
        self.returns: list[float] = []

    @property
    def baseline(self) -> float:
        return math.fsum(self.returns) / len(self.returns) if self.returns else 0.0

    def observe(self, r: float) -> None:
        self.returns.append(r)


def _episode_seeds(config: TrainConfig, stage: str) -> list[int]:
    root = np.random.SeedSequence([config.seed, STAGES.index(stage)])
    return [int(s.generate_state(1)[0]) for s in root.spawn(config.episodes)]


@dataclass
class StageResult:
    stage: str
    params: Params
    curve: list[dict]
    best_makespan: float | None = None
    best_assignment: Assignment | None = None
    encoder_invocations: int = 0
    final_loss: float | None = None


class GlobalUpdate:
    """Device-agnostic part of one batched update shared by every rank:
    the running-mean baseline over ALL previous returns of all ranks
    (training.py:65-78, 196-198), alpha_e = (mk_e + baseline) / B_g, and the
    single collective: allreduce(SUM) of [flat grad | sum of local returns]."""

    def __init__(self, n_params: int, batch_size: int, world: int = 1, group=None,
                 device="cuda"):
        import torch

        self.world, self.group = world, group
        self.Bg = batch_size * world
        self.gbuf = torch.zeros(n_params + 1, dtype=torch.float64, device=device)
        self.grad = self.gbuf[:n_params]
        self.ret_sum = torch.zeros(1, dtype=torch.float64, device=device)
        self.count = 0

    def baseline(self):
        import torch

        return self.ret_sum / self.count if self.count else torch.zeros_like(self.ret_sum)

    def alpha(self, makespan, out, n_global: int | None = None):
        """alpha_e = -advantage_e / B_g with advantage_e = -mk_e - baseline
        (``n_global`` episodes in this update, B_g unless it is a short last
        batch)."""
        import torch

        return torch.add(makespan, self.baseline(), out=out).mul_(1.0 / (n_global or self.Bg))

    def finish(self, makespan, n_global: int | None = None):
        """Append sum of local returns, allreduce, advance the baseline.
        ``makespan`` holds this rank's valid episodes only (may be empty)."""
        import torch
        import torch.distributed as dist

        if makespan.numel():
            torch.sum(makespan, dim=0, keepdim=True, out=self.gbuf[-1:]).neg_()
        else:
            self.gbuf[-1:].zero_()
        if self.world > 1:
            dist.all_reduce(self.gbuf, op=dist.ReduceOp.SUM, group=self.group)
        self.ret_sum += self.gbuf[-1:]
        self.count += n_global or self.Bg


class BatchedTrainer:
    """B episodes per update on one GPU; ``world`` > 1 shards episodes over
    ranks (torch.distributed NCCL group) with one allreduce per update."""

    def __init__(self, ctx: PolicyContext, params, config: TrainConfig, batch_size: int = 1024,
                 world: int = 1, rank: int = 0, group=None, stage: str = "sim_rl",
                 executor=None, teacher=None):
        import torch

        self.ctx = ctx
        self.config = config
        self.B = int(batch_size)
        self.world, self.rank, self.group = world, rank, group
        self.stage = stage
        self.executor = executor
        # imitation teacher: None / CriticalPathRule run in the kernel; any
        # other select / place object is stepped on the host (FORCED replay)
        self.teacher = None if teacher is None or is_native_teacher(teacher) else teacher
        self.Bg = self.B * world
        self.flat = ctx.flat_params(params).clone()
        self.upd = GlobalUpdate(ctx.layout.size, self.B, world, group)
        self.grad = self.upd.grad
        self.alpha = torch.empty(self.B, dtype=torch.float64, device="cuda")
        self.updates = 0
        self.lr_sched = LinearSchedule(config.lr0, config.lr1, config.episodes)
        self.eps_sched = LinearSchedule(config.epsilon0, 0.0, config.episodes)
        self.out = None
        # failed rollouts are detected without a host sync inside the step: a
        # sticky device flag (count of failed episodes) masks every later SGD
        # update, and its pinned host copy is checked -- raising -- at the
        # next step once it has landed, or by check() (blocking)
        self.failed = torch.zeros(1, dtype=torch.int32, device="cuda")
        self._failed_host = torch.zeros(1, dtype=torch.int32, pin_memory=True)
        self._failed_ev = None

    def load_flat(self, flat):
        self.flat.copy_(flat)

    def params(self) -> Params:
        return self.ctx.layout.unflatten(self.flat.cpu().numpy())

    def launches_per_step(self) -> int:
        pc = self.ctx.config
        n_enc = 1 if pc.shared_encoder else 2
        # encode (K+1) + rollout + reduce (2) + alpha/baseline (torch ops: not ours)
        # + backward (head 2 + outer 2 + small 1 + per (enc, round) 3 (+copy)) + sgd
        per_round = n_enc * pc.k_rounds * 4 - n_enc
        return self.ctx.encode_launches() + 1 + 2 + 5 + per_round + 1

    def check(self, block: bool = True) -> None:
        """Raise if a rollout of an earlier step failed (the parameters were
        left at their value before that step: its SGD update was masked)."""
        ev = self._failed_ev
        if ev is None or (not block and not ev.query()):
            return
        ev.synchronize()
        nbad = int(self._failed_host[0])
        if nbad:
            raise RuntimeError(f"rollout failed for {nbad} episode(s); parameters kept at their "
                               "value before the failing update")

    def local_count(self, n_global: int) -> int:
        """Episodes of a (possibly short) update of ``n_global`` episodes that
        fall on this rank: global index u*B_g + rank*B + b, b < B."""
        return max(0, min(self.B, n_global - self.rank * self.B))

    def step(self, seed: int, out=None, kernel_events=None, record=False,
             n_global: int | None = None):
        """One update over B local episodes (``n_global`` < B_g: a short last
        batch of exactly that many episodes across the ranks; a rank with no
        episode still joins the allreduce).  Returns host stats when
        ``record`` (makespans, advantages, epsilon, lr, per-episode loss for
        imitation) — that needs a sync."""
        import torch

        ctx = self.ctx
        self.check(block=False)
        ng = self.Bg if n_global is None else int(n_global)
        if not 0 < ng <= self.Bg:
            raise ValueError(f"n_global must be in 1..{self.Bg}")
        Bl = self.local_count(ng)
        ep0 = self.upd.count  # global episodes before this batch
        eps = 0.0 if self.stage == "imitation" else self.eps_sched.value(ep0)
        lr = self.lr_sched.value(ep0)
        if out is None:
            out = self.out = self.out or ctx.alloc_batch(
                self.B, grad=True, trace_steps=self.stage == "imitation")
        ctx.prepare(self.flat)
        if kernel_events is not None:
            kernel_events[0].record()
        mode = "teacher" if self.stage == "imitation" else "sample"
        forced = None
        if self.stage == "imitation" and self.teacher is not None and Bl:
            mode = "forced"
            forced = torch.from_numpy(
                teacher_actions(ctx.graph, ctx.cluster, self.teacher, Bl)).cuda()
        if Bl:
            ctx.rollout_batch(self.flat, Bl, eps, seed, mode=mode, forced=forced, grad=True,
                              out=out, episode_base=self.rank * self.B, prepare=False,
                              simulate=self.executor is None, strategy=self.config.strategy)
        if kernel_events is not None:
            kernel_events[1].record()
        if self.executor is not None and Bl and hasattr(self.executor, "batch"):
            # Stage III with a batched executor: the whole batch in one call
            mk = self.executor.batch(ctx, out.assign[:Bl])
        elif self.executor is not None and Bl:
            # Stage III: rewards from an external executor (host callable)
            assign = out.assign[:Bl].cpu().numpy()
            mkl = [float(self.executor(ctx.graph, Assignment(tuple(int(x) for x in a))))
                   for a in assign]
            mk = torch.tensor(mkl, dtype=torch.float64, device="cuda")
        else:
            mk = out.makespan[:Bl]
        if Bl:  # no host sync: counted on the device, SGD masked, raised later
            self.failed += (out.status[:Bl] != 0).sum(dtype=torch.int32)
        if record and Bl and bool((out.status[:Bl] != 0).any()):
            st = out.status[:Bl].cpu().numpy()
            raise RuntimeError(f"rollout failed for {int((st != 0).sum())} of {Bl} episodes "
                               f"(status codes {sorted(set(st.tolist()) - {0})})")
        # alpha_e = -adv_e / n_global, adv_e = -mk_e - baseline
        if record:
            base_host = float(self.upd.baseline().item())
        alpha = self.alpha[:Bl]
        if self.stage == "imitation":
            alpha.fill_(-1.0 / ng)
            beta = 0.0
        else:
            self.upd.alpha(mk, alpha, ng)
            beta = -self.config.entropy_weight / ng
        if Bl:
            ctx.reduce_gradient(out.grad_rows, out.grad_ep, out.assign, alpha, beta, Bl,
                                self.grad)
        else:
            self.grad.zero_()
        self.upd.finish(mk, ng)
        N.check(N.lib().fp_sgd_step_masked(N.ptr(self.flat), N.ptr(self.grad),
                                           ctypes.c_int64(self.grad.numel()), ctypes.c_double(lr),
                                           N.ptr(self.failed), N.stream_ptr()))
        self._failed_host.copy_(self.failed, non_blocking=True)
        if self._failed_ev is None:
            self._failed_ev = torch.cuda.Event()
        self._failed_ev.record()
        self.updates += 1
        if record:
            mkh = mk.cpu().numpy()
            rec = {"makespan": mkh, "advantage": -mkh - base_host, "epsilon": eps, "lr": lr,
                   "assign": out.assign[:Bl].cpu().numpy()}
            if out.step_lp is not None:
                # imitation loss of each episode: -sum of its 2n log-probs
                # (training.py:144-146; np.sum of the concatenated [1, 2n] row)
                lp = out.step_lp[:Bl].cpu().numpy().reshape(Bl, 1, -1)
                rec["loss"] = [float(-np.sum(lp[b])) for b in range(Bl)]
            return rec
        return None


def measure_teacher_agreement(ctx: PolicyContext, params, teacher, rollouts: int = 100,
                              seed: int = 0) -> float:
    """Fraction of teacher-forced steps where the policy's greedy action
    matches the teacher's, select and place counted separately
    (training.py:162-178).  All ``rollouts`` episodes run as one teacher-mode
    batch on the GPU (episode k keyed by seed + k, as the reference's seeds)."""
    if rollouts <= 0:
        return 1.0
    if teacher is None or is_native_teacher(teacher):
        rb = ctx.rollout_batch(params, rollouts, 0.0, seed, mode="teacher", simulate=False,
                               trace_steps=True)
    else:  # duck-typed teacher: host-stepped actions, replayed in FORCED mode
        acts = teacher_actions(ctx.graph, ctx.cluster, teacher, rollouts)
        rb = ctx.rollout_batch(params, rollouts, 0.0, seed, mode="forced", forced=acts,
                               simulate=False, trace_steps=True)
    st = rb.status.cpu().numpy()
    if (st != 0).any():
        raise RuntimeError(f"teacher rollout failed (status {sorted(set(st.tolist()))})")
    vd = rb.step_vd.cpu().numpy()
    am = rb.step_argmax.cpu().numpy()
    agree = int((am[..., 0] == vd[..., 0]).sum()) + int((am[..., 1] == vd[..., 1]).sum())
    total = 2 * vd.shape[0] * vd.shape[1]
    return agree / total if total else 1.0


def _stage(stage: str, graph, cluster, config: TrainConfig, pconfig: PolicyConfig, params,
           context=None, batch_size: int = 1, executor=None, world=1, rank=0, group=None,
           teacher=None):
    ctx = context or PolicyContext(graph, cluster, pconfig)
    start_enc = ctx.encode_count
    tr = BatchedTrainer(ctx, params, config, batch_size, world, rank, group, stage, executor,
                        teacher=teacher)
    seeds = _episode_seeds(config, stage)
    curve = []
    best_mk, best_assign = None, None
    n_updates = (config.episodes + tr.Bg - 1) // tr.Bg
    final_loss = None
    for u in range(n_updates):
        # exactly config.episodes episodes: the last update may be short
        ng = min(tr.Bg, config.episodes - u * tr.Bg)
        st = tr.step(seed=seeds[u * tr.Bg], record=True, n_global=ng)
        for b in range(len(st["makespan"])):
            idx = u * tr.Bg + rank * tr.B + b
            mk = float(st["makespan"][b])
            row = {"index": idx, "makespan_ms": mk, "advantage": float(st["advantage"][b]),
                   "epsilon": st["epsilon"], "lr": st["lr"]}
            if stage == "imitation":
                row["advantage"] = 0.0
                row["loss"] = final_loss = st["loss"][b]
            curve.append(row)
            if best_mk is None or mk < best_mk:
                best_mk = mk
                best_assign = Assignment(tuple(int(x) for x in st["assign"][b]), "doppler")
    tr.check()
    out_params = tr.params()
    if isinstance(params, dict):  # keep the caller's dict in sync (reference mutates in place)
        for k, v in out_params.items():
            if k in params and hasattr(params[k], "data"):
                params[k].data[...] = v.data
    return StageResult(stage, params if isinstance(params, dict) else out_params, curve,
                       best_makespan=None if stage == "imitation" else best_mk,
                       best_assignment=None if stage == "imitation" else best_assign,
                       encoder_invocations=ctx.encode_count - start_enc,
                       final_loss=final_loss)


def imitation_stage(graph, cluster, config, pconfig, params, teacher=None, context=None,
                    batch_size: int = 1, **kw):
    """Teacher-forced behavioural cloning (training.py:129-155): CriticalPathRule
    (the default) runs inside the rollout kernel; any other teacher with the
    reference's select / place interface is stepped on the host per episode
    and its actions replayed in FORCED mode."""
    if teacher is not None and not is_native_teacher(teacher):
        kw["teacher"] = teacher
    return _stage("imitation", graph, cluster, config, pconfig, params, context, batch_size, **kw)


def sim_rl_stage(graph, cluster, config, pconfig, params, context=None, batch_size: int = 1,
                 **kw):
    """Policy gradient with the clean GPU simulator as reward (training.py:219-232)."""
    return _stage("sim_rl", graph, cluster, config, pconfig, params, context, batch_size, **kw)


def system_rl_stage(graph, cluster, executor, config, pconfig, params, context=None,
                    batch_size: int = 1, **kw):
    """Policy gradient with rewards from an executor (training.py:235-248)."""

    def safe(g, a):
        try:
            return float(executor(g, a))
        except Exception as exc:  # noqa: BLE001 — reference wraps every failure
            raise RuntimeError(f"executor failed: {exc}") from exc

    if hasattr(executor, "batch"):  # a batched executor scores the whole batch at once
        def safe_batch(ctx, assign):
            try:
                return executor.batch(ctx, assign)
            except Exception as exc:  # noqa: BLE001
                raise RuntimeError(f"executor failed: {exc}") from exc
        safe.batch = safe_batch

    return _stage("system_rl", graph, cluster, config, pconfig, params, context, batch_size,
                  executor=safe, **kw)


class SimulatorExecutor:
    """Executor stand-in: the GPU simulator with per-call jitter seeds
    (training.py:81-102; reference-exact host jitter tables)."""

    def __init__(self, cluster: ClusterSpec, strategy: str = "fifo", jitter_sigma: float = 0.1,
                 base_seed: int = 0):
        if jitter_sigma > 0:
            cluster = ClusterSpec.from_dict({**cluster.to_dict(), "jitter_sigma": jitter_sigma})
        self.cluster = cluster
        self.strategy = strategy
        self.base_seed = base_seed
        self._calls = itertools.count()

    def __call__(self, graph: DataflowGraph, assignment) -> float:
        seed = self.base_seed + next(self._calls)
        prob = self._problem(graph)
        import torch
        a = torch.tensor([list(assignment)], dtype=torch.int32, device="cuda")
        jit = prob.jitter_table(seed)
        jt = torch.from_numpy(jit).cuda() if jit is not None else None
        out = prob.simulate(a, self.strategy, jitter=jt)
        if int(out["status"][0]) != 0:
            raise RuntimeError("simulation deadlocked")
        return float(out["makespan"][0])

    def _problem(self, graph: DataflowGraph):
        from .simulate import SimProblem

        prob = getattr(self, "_prob", None)
        if prob is None or prob.graph is not graph:
            self._prob = prob = SimProblem(graph, self.cluster)
        return prob

    def batch(self, ctx, assign):
        """Makespans of a device batch of assignments [B, n] in one launch:
        episode i gets the i-th next seed of the call stream, exactly as B
        successive calls would (per-task jitter factors from the reference's
        host libm recipe, one table per episode)."""
        import torch

        prob = self._problem(ctx.graph)
        B = assign.shape[0]
        seeds = [self.base_seed + next(self._calls) for _ in range(B)]
        jt = None
        if self.cluster.jitter_sigma > 0:
            jt = torch.from_numpy(np.stack([prob.jitter_table(sd) for sd in seeds])).cuda()
        out = prob.simulate(assign, self.strategy, jitter=jt)
        if bool((out["status"] != 0).any()):
            raise RuntimeError("simulation deadlocked")
        return out["makespan"]


SIDECAR_SUFFIX = ".sidecar.json"


def save_checkpoint(path, params, pconfig: PolicyConfig, config: TrainConfig,
                    norm_stats: dict | None = None) -> None:
    path = Path(path)
    save_params(params, path)
    sidecar = {"policy": pconfig.to_dict(), "train": config.to_dict(),
               "feature_norm": norm_stats or {},
               "epsilon": {"v0": config.epsilon0, "v1": 0.0, "total": config.episodes}}
    Path(str(path) + SIDECAR_SUFFIX).write_text(json.dumps(sidecar, indent=2, sort_keys=True) + "\n")


def load_checkpoint(path):
    path = Path(path)
    params = load_params(path)
    sc = Path(str(path) + SIDECAR_SUFFIX)
    sidecar = json.loads(sc.read_text()) if sc.exists() else {}
    pconfig = PolicyConfig.from_dict(sidecar.get("policy", {}))
    want = param_shapes(pconfig)
    if set(want) != set(params):
        raise ValueError(f"checkpoint does not match policy config: "
                         f"{sorted(set(want) ^ set(params))}")
    for name, shape in want.items():
        if params[name].shape != shape:
            raise ValueError(f"checkpoint tensor {name} has shape {params[name].shape}, "
                             f"expected {shape}")
    return params, pconfig, sidecar
