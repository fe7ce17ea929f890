"""Throughput bench for the DOPPLER rollout hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload ffnn]
                    [--batch B] [--mode rollout|train] [--impl ours|reference]

One step = one pass of the hot path over one batch: encode the graph for the
parameter snapshot (GNN + head tables), run B SEL/PLC episodes (epsilon 0.2
Philox sampling) each scored by the work-conserving simulator (config 2 of
BASELINE.json: FFNN graph, 8 simulated devices, 1024 episodes per GPU).
``--mode train`` adds the Stage-II REINFORCE update (reduction, backward,
NCCL allreduce of the gradient, SGD).  N>1: one process per GPU (torchrun),
episodes sharded (weak scaling), time = max over ranks.

``--impl reference`` times the REFERENCE itself on all host cores: the
``flowplace`` package built by ``oracle/build_ref.sh`` into ``oracle/_ref``
(its Cython simulator core), one process per core looping exactly the calls
of its trainer (``training.py:193-194``: ``PolicyContext.rollout`` +
``exec_time``; ``--mode train`` runs ``sim_rl_stage``, i.e. adds the tape
backward and SGD).  Without ``oracle/_ref`` it falls back to the oracle port
(numpy rollout + the C restatement of ``_simcore.pyx``), ``kind: "port"``.
The default workload is BASELINE config 3's per-GPU share: the Llama-block
graph, 8 simulated devices, 1024 episodes per GPU (8192 at 8 GPUs).
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "simulated placement episodes/sec"
UNIT = "episodes/s"
EPSILON = 0.2


def workload(name: str):
    from paper_2505_23131_b200 import builders
    from paper_2505_23131_b200.cluster import ClusterSpec
    if name == "ffnn":
        return (builders.build_ffnn(8, 4, 16, 4, 2),
                ClusterSpec.uniform(8, rate=1e6, bandwidth=1e5, comm_factor=4),
                "FFNN build_ffnn(8,4,16,4,2): 64 ops / 92 edges, 8 devices")
    if name == "chainmm":
        return (builders.build_chainmm(64, 2),
                ClusterSpec.uniform(4, rate=1e6, bandwidth=1e5, comm_factor=4),
                "ChainMM build_chainmm(64,2): 60 ops / 80 edges, 4 devices")
    if name == "llama_block":
        return (builders.build_llama_block(), ClusterSpec.uniform(8, rate=1e9, bandwidth=1e7),
                "Llama-7B block (shard_grid 2): 208 ops / 324 edges, 8 devices")
    if name == "llama_layer":
        return (builders.build_llama_layer(), ClusterSpec.uniform(8, rate=1e9, bandwidth=1e7),
                "Llama-7B layer + LM head (shard_grid 2): 248 ops / 392 edges, 8 devices")
    if name.startswith("dag"):
        n = int(name[3:].replace("k", "000"))
        return (builders.sparse_dag(n, seed=0), ClusterSpec.uniform(8, rate=1e9, bandwidth=1e7),
                f"sparse DAG {n} ops, 8 devices")
    raise SystemExit(f"unknown workload {name}")


# --------------------------------------------------------------------------- CPU
REF_DIR = ROOT / "oracle" / "_ref"


def ref_available() -> bool:
    return (REF_DIR / "flowplace" / "policy.py").exists()


def _ref_worker(args):
    """The reference's own episodes on one core until the deadline:
    PolicyContext.rollout + exec_time (training.py:193-194), or sim_rl_stage
    chunks (rollout + reward + tape backward + SGD) in train mode."""
    wl, seed0, deadline, train, per_step = args
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    os.environ.pop("FLOWPLACE_SIM_BACKEND", None)
    from flowplace import graph as RG
    from flowplace import simulate as RS
    from flowplace.cluster import ClusterSpec as RC
    from flowplace.policy import PolicyConfig as RPC, PolicyContext as RPX, init_policy_params as rinit
    from flowplace.training import TrainConfig as RTC, sim_rl_stage
    from paper_2505_23131_b200.graph import graph_to_dict
    assert RS.backend_name() == "cython", RS.backend_name()
    g, cl, _ = workload(wl)
    rg = RG.graph_from_dict(graph_to_dict(g))
    rc = RC.from_dict(cl.to_dict())
    pc = RPC(hidden=32, k_rounds=2, mp_mode="per_step" if per_step else "per_episode")
    params = rinit(pc, seed=0)
    ctx = RPX(rg, rc, pc)
    done = 0
    t0 = time.perf_counter()
    while time.perf_counter() < deadline or done == 0:
        if train:
            sim_rl_stage(rg, rc, RTC(episodes=1, seed=seed0 + done), pc, params, context=ctx)
        else:
            a, _ = ctx.rollout(params, epsilon=EPSILON, seed=seed0 + done)
            RS.exec_time(rg, a, rc, "fifo", seed=0, features=ctx.features)
        done += 1
    return done, time.perf_counter() - t0


def _port_worker(args):
    """Reference-algorithm episodes (the oracle port) on one core."""
    wl, seed0, deadline, train, per_step = args
    from oracle import policy as OP
    from oracle import sim as osim
    from paper_2505_23131_b200.params import init_policy_params
    from paper_2505_23131_b200.policy import PolicyConfig
    g, cl, _ = workload(wl)
    pc = PolicyConfig(mp_mode="per_step" if per_step else "per_episode")
    params = init_policy_params(pc, seed=0)
    ctx = OP.Ctx(g, cl, pc.hidden, pc.k_rounds, pc.leaky_slope, pc.shared_encoder)
    packed = osim.pack(g, [0] * len(g), cl, ctx.f, "fifo", 0)
    done = 0
    t0 = time.perf_counter()
    while time.perf_counter() < deadline or done == 0:
        if train:
            _, ro = OP.rl_gradients(params, ctx, EPSILON, -1.0, 1e-2, mode="uniform",
                                    seed=seed0, episode=done)
        else:
            ro = OP.rollout(OP.leaves(params), ctx, EPSILON, mode="uniform", seed=seed0,
                            episode=done, per_step=per_step)
        osim.sim_batch(packed, np.asarray([ro["assign"]], dtype=np.int32))
        done += 1
    return done, time.perf_counter() - t0


def _cpu_worker(args):
    return (_ref_worker if ref_available() else _port_worker)(args)


_POOL = None


def _pool(procs: int):
    """One worker process per core, single-threaded BLAS (spawned with the
    env set, so numpy's BLAS never starts extra threads); reused across
    steps."""
    global _POOL
    if _POOL is None:
        for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
            os.environ[k] = "1"
        _POOL = mp.get_context("spawn").Pool(procs)
    return _POOL


def cpu_throughput(wl: str, seconds: float, procs: int, train: bool = False,
                   per_step: bool = False):
    pool = _pool(procs)
    # every worker imports its stack first (untimed), then runs to a shared deadline
    pool.map(_warm_worker, [(wl, per_step)] * procs)
    deadline = time.perf_counter() + seconds
    res = pool.map(_cpu_worker, [(wl, 1000 + 7919 * i, deadline, train, per_step)
                                 for i in range(procs)])
    eps = sum(r[0] for r in res)
    wall = max(r[1] for r in res)
    return eps / wall, eps, wall


def _warm_worker(args):
    wl, per_step = args
    _cpu_worker((wl, 0, 0.0, False, per_step))
    return True


def cpu_kind() -> str:
    return "reference" if ref_available() else "port"


def cpu_sample_desc(eps_done: int, wall: float, procs: int, train: bool = False) -> str:
    if ref_available():
        what = ("flowplace reference (oracle/_ref, Cython simulator core): " +
                ("sim_rl_stage, one episode per call (rollout + exec_time + backward + SGD)"
                 if train else "PolicyContext.rollout + exec_time per episode"))
    else:
        what = "oracle port (numpy rollout + C simulator)"
    return f"{eps_done} episodes in {wall:.1f}s across {procs} processes, {what}"


def bench_config(args, world: int, desc: str) -> dict:
    """The config both arms report (same keys, so the driver can pair them)."""
    return {"workload": desc, "episodes_per_gpu": args.batch,
            "global_batch": args.batch * world, "mode": args.mode, "epsilon": EPSILON,
            "policy": f"hidden 32, K 2, {args.mp_mode}" + (
                "" if args.encoder == "dmma" else f", {args.encoder} encoder"),
            "outputs": ("assignments, makespans + per-step trace (log-probs, entropies, argmax)"
                        if args.full_outputs else "assignments + makespans"),
            "parallelism": f"episode-dp{world}",
            "l2": "GPU arm: flushed between timed steps (256 MiB write); e2e: steps pipelined "
                  "(H2D of the parameters and D2H of the results on side streams, double-buffered), "
                  "L2 evicted every step by a "
                  "128 MiB device-to-device copy (copy engine, 256 MiB through L2) on the side "
                  "stream"}


# --------------------------------------------------------------------------- clocks
class Clocks:
    def __init__(self, path: Path):
        self.path = path
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()

    def summary(self, gpu_index: int):
        try:
            rows = [r.split(", ") for r in self.path.read_text().strip().splitlines()]
        except OSError:
            return None
        rows = [r for r in rows if len(r) >= 9 and r[0].strip() == str(gpu_index)]
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].strip() == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(rows[0][2]) if rows[0][2].strip().replace(".", "").isdigit()
                else None, "reasons": reasons, "samples": len(rows)}


# --------------------------------------------------------------------------- GPU
def _episode_rates(g, assign: np.ndarray, episodes_per_s: float) -> dict:
    """Decisions/s and simulated WC events/s from the last timed
    batch: an episode makes n SEL+PLC decisions and its simulation runs one
    exec per non-entry vertex plus one transfer per (vertex, other consumer
    device) -- 2 events (beg, end) per task."""
    c = g.csr()
    n = len(g)
    src = np.repeat(np.arange(n), np.diff(c["succ_indptr"]))
    dst = c["succ_indices"].astype(np.int64)
    B = assign.shape[0]
    a = assign.astype(np.int64)
    cons = np.zeros((B, n), dtype=np.int64)
    for e in range(len(src)):  # device bitmask of each vertex's consumers
        cons[:, src[e]] |= np.left_shift(1, a[:, dst[e]])
    cons &= ~np.left_shift(1, a)
    nonentry = c["is_entry"] == 0
    bits = np.zeros_like(cons)
    x = cons.copy()
    while x.any():
        bits += x & 1
        x >>= 1
    tasks = int(nonentry.sum()) + bits[:, nonentry].sum(axis=1)
    return {"decisions_per_s": episodes_per_s * n,
            "sim_tasks_per_episode": float(tasks.mean()),
            "sim_events_per_s": episodes_per_s * 2 * float(tasks.mean())}


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # FP_BENCH_DIST_BACKEND=gloo (+ ranks sharing a GPU) exercises the
    # multi-rank code path on a one-GPU box; the driver's runs use NCCL
    backend = os.environ.get("FP_BENCH_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    from paper_2505_23131_b200.params import init_policy_params
    from paper_2505_23131_b200.policy import PolicyConfig, PolicyContext

    g, cl, desc = workload(args.workload)
    n = len(g)
    pc = PolicyConfig(mp_mode=args.mp_mode)
    params = init_policy_params(pc, seed=0)
    ctx = PolicyContext(g, cl, pc)
    if args.encoder != "dmma":
        ctx.set_encoder(args.encoder)
    B = args.batch
    train = args.mode == "train"
    trainer = None
    if train:
        from paper_2505_23131_b200.training import BatchedTrainer, TrainConfig
        trainer = BatchedTrainer(ctx, params, TrainConfig(episodes=10 ** 6), batch_size=B,
                                 world=world, rank=rank)
    flat = ctx.flat_params(params)
    out = ctx.alloc_batch(B, grad=train, trace_steps=args.full_outputs)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    ep_base = rank * B

    def step(i):
        seed = 0x5EED0000 + i
        if train:
            trainer.step(seed=seed, out=out)
        else:
            ctx.rollout_batch(flat, B, EPSILON, seed, episode_base=ep_base, out=out)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()

    # ---- device-timed steps (L2 flushed between steps, outside the events) ----
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    clk = Clocks(ROOT / "gpurun_out" / f"clocks_rank{rank}.csv") if rank == 0 else None
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if clk:
        clk.__enter__()
        time.sleep(0.3)
    from paper_2505_23131_b200 import _native as N
    # per_step: an event pair around every aggregation launch (its own stream);
    # not in per_episode, where the events would sit between PDL-chained kernels
    N.agg_timer(args.mp_mode == "per_step")
    for i in range(args.steps):
        flush.fill_(float(i))
        ev[i][0].record(stream)
        if train:
            trainer.step(seed=0x7000 + i, out=out, kernel_events=kev[i])
        else:
            ctx.prepare(flat)
            kev[i][0].record(stream)
            ctx.rollout_batch(flat, B, EPSILON, 0x7000 + i, episode_base=ep_base, out=out,
                              prepare=False)
            kev[i][1].record(stream)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    agg_ms, agg_launches = N.agg_timer_read()
    N.agg_timer(False)
    if world > 1:
        dist.barrier()
    if clk:
        clk.__exit__()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    kern_ms = [a.elapsed_time(b) for a, b in kev]
    tot = torch.tensor([sum(step_ms)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    total_ms = float(tot.item())
    ms_per_step = total_ms / args.steps
    value = B * world * args.steps / (total_ms / 1e3)
    st = out.status.cpu().numpy()
    assert (st == 0).all(), "episode failures in the timed region"

    # ---- end-to-end through the public API with host buffers ----
    # Every step: H2D of its parameters from pinned host memory, the public
    # rollout_batch / trainer.step call, D2H of its assignments + makespans
    # into pinned host memory.  Steps are pipelined the way a serving loop
    # would run them: the D2H copies go on a side stream and the device
    # outputs are double-buffered, so step i's copies overlap step i+1's
    # kernels; the whole run is timed once on the host clock (synchronized on
    # both sides), no per-step device timing.
    host_params = torch.from_numpy(ctx.layout.flatten(params)).pin_memory()
    host_assign = [torch.empty((B, n), dtype=torch.int32).pin_memory() for _ in range(2)]
    host_mk = [torch.empty(B, dtype=torch.float64).pin_memory() for _ in range(2)]
    dev_params = [torch.empty_like(flat) for _ in range(2)]
    outs = [out, ctx.alloc_batch(B, grad=train, trace_steps=args.full_outputs)]
    copy_stream = torch.cuda.Stream()
    h2d_stream = torch.cuda.Stream()
    h2d_ev = [torch.cuda.Event() for _ in range(2)]
    done_ev = [torch.cuda.Event() for _ in range(2)]
    free_ev = [torch.cuda.Event() for _ in range(2)]

    def e2e_step(i):
        sl = i % 2
        comp = torch.cuda.current_stream()
        # H2D of this step's parameters on its own stream, double-buffered, so
        # it overlaps the previous step's kernels (step i-2 must be done with
        # the buffer); the step's kernels wait for it
        with torch.cuda.stream(h2d_stream):
            if i >= 2:
                h2d_stream.wait_event(done_ev[sl])
            dev_params[sl].copy_(host_params, non_blocking=True)
            h2d_ev[sl].record(h2d_stream)
        comp.wait_event(h2d_ev[sl])
        if i >= 2:
            comp.wait_event(free_ev[sl])  # step i-2's results are on the host
        if train:
            trainer.load_flat(dev_params[sl])
            trainer.step(seed=0x9000 + i, out=outs[sl])
        else:
            ctx.rollout_batch(dev_params[sl], B, EPSILON, 0x9000 + i, episode_base=ep_base,
                              out=outs[sl])
        done_ev[sl].record(comp)
        with torch.cuda.stream(copy_stream):
            copy_stream.wait_event(done_ev[sl])
            host_assign[sl].copy_(outs[sl].assign, non_blocking=True)
            host_mk[sl].copy_(outs[sl].makespan, non_blocking=True)
            free_ev[sl].record(copy_stream)
            # evict L2 while the next step runs: a 128 MiB -> 128 MiB device
            # copy (copy engine, 256 MiB through L2) keeps the SMs for the
            # measured steps (a fill kernel competed with them for SM slots)
            flush[: flush.numel() // 2].copy_(flush[flush.numel() // 2:])

    for i in range(args.warmup):
        e2e_step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for i in range(args.steps):
        e2e_step(args.warmup + i)
    torch.cuda.synchronize()
    e2e_ms = [(time.perf_counter() - t0) * 1e3]
    assert bool((outs[0].status == 0).all()) and bool((outs[1].status == 0).all())
    e2e_t = torch.tensor([sum(e2e_ms)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = B * world * args.steps / (float(e2e_t.item()) / 1e3)

    if rank == 0:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (
            ROOT / "MEASURED_PEAKS.json").exists() else {}
        peak = peaks.get("hbm_gbs", 6650.0)
        kms = float(np.mean(kern_ms))
        # algorithmic bytes of one rollout launch: per episode
        # 4n (assign out) + 12 (makespan, status out); per launch the graph
        # CSR + policy tables read once: (n+1)*8 + E*8 + 16n + n*8 + 2*n*h*8
        E = len(g.edges)
        h = pc.hidden
        per_ep = 4 * n + 12
        per_launch = (n + 1) * 8 + E * 8 + 16 * n + 8 * n + 2 * n * h * 8
        alg = B * per_ep + per_launch
        if train:  # REINFORCE decision records written (grad_rec_stride doubles per step)
            alg += B * n * ctx.grad_rec_stride() * 8
        per_step = args.mp_mode == "per_step"
        K = pc.k_rounds
        prep_launches = ctx.encode_launches()
        # GNN aggregation kernel (north star: >= 60% of HBM), timed on its own
        # launching stream over the timed region (fp_agg_timer_*).  Algorithmic
        # bytes per launch and encoder: every row's P (gathered; each row is
        # needed once), Q and agg rows once -- 3 x 8h B per row in fp64, fp32
        # P/Q + bf16 hi/lo agg planes (3 x 4h B) for the tc encoder -- plus
        # the message CSR (ptr 4 B per vertex, source 4 B + edge scalar 8 B per
        # message), read once per encoder
        rows = B * n if per_step else n
        M = 2 * len(g.edges)
        row_b = 3 * (4 if args.encoder == "tc" else 8) * h
        n_enc = 1 if pc.shared_encoder else 2
        agg_alg = n_enc * (rows * row_b + (n + 1) * 4 + M * 12)
        agg = None
        if agg_launches:
            agg_kms = agg_ms / agg_launches
            agg_ach = agg_alg / (agg_kms * 1e-3) / 1e9
            agg = {"kernel": "gnn_agg_staged_kernel" if per_step else "gnn_agg_kernel",
                   "rows_per_encoder": rows, "encoders": n_enc,
                   "alg_bytes_per_launch": agg_alg, "kernel_ms": agg_kms,
                   "launches_timed": agg_launches, "achieved": agg_ach, "peak": peak,
                   "unit": "GB/s", "frac": agg_ach / peak}
        if per_step:
            launches = prep_launches + 1 + n * (2 + 2 * K) + 3
        else:
            launches = prep_launches + 1
        achieved = alg / (kms * 1e-3) / 1e9
        # DRAM traffic and executed instructions of this very kernel and config,
        # from the ncu capture of the same bench command committed this round
        # (tools/roofline_capture.sh -> profiles/r2/rollout_ncu.json)
        traffic, ncu_rec = None, None
        tpath = ROOT / "profiles" / "r2" / "rollout_ncu.json"
        if tpath.exists() and not per_step:
            ncu_rec = json.loads(tpath.read_text()).get(
                f"{args.workload}/{'train' if train else 'rollout'}/B{B}")
            if ncu_rec:
                traffic = ncu_rec["dram_bytes_read"] + ncu_rec["dram_bytes_write"]
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64" if args.encoder == "dmma" else "f64 (node MLPs: split-bf16 tcgen05, f32 accumulate)",
            "data": "synthetic (builder graph; random-init policy seed 0; Philox episodes)",
            "config": bench_config(args, world, desc),
            "e2e": {"value": e2e_value, "unit": UNIT,
                    "h2d_bytes_per_step": int(host_params.numel() * 8),
                    "d2h_bytes_per_step": int(B * n * 4 + B * 8)},
            "gpu_launches": args.steps * (launches if not train else
                                          trainer.launches_per_step()),
            "roofline": {"bound": "hbm", "kernel": ("per_step rollout (batched aggregation)"
                                                    if per_step else "rollout_kernel")
                         if not train else "rollout_kernel(grad)", "achieved": achieved,
                         "peak": peak,
                         "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                         "kernel_ms": kms, "alg_bytes_per_launch": alg,
                         "note": ("B x n batched encodes per step; per-launch aggregation "
                                  "bytes summed over the whole rollout" if per_step else
                                  "latency-bound: each episode is a dependent chain of n "
                                  "decisions + the overlapped simulation (DESIGN.md section 4); "
                                  "GNN aggregation roofline: --mp-mode per_step, "
                                  "profiles/r2/final/ncu_agg_staged_*"),
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback"},
        }
        if agg:
            if per_step:
                # per_step: the aggregation kernel IS the HBM-bound kernel of
                # the step (B x n rows per launch); its own roofline heads the
                # line, the rollout-wide figure stays beside it
                blended = line["roofline"]
                line["roofline"] = dict(agg, bound="hbm", traffic=None,
                                        peak_source=blended["peak_source"],
                                        note="gnn aggregation kernel, event-timed per launch "
                                             "over the timed region; algorithmic bytes = "
                                             "P, Q, agg rows once + the message CSR",
                                        rollout=blended)
            else:
                line["roofline"]["aggregation"] = agg
        line["rates"] = _episode_rates(g, out.assign.cpu().numpy(), value)
        if clk:
            line["clocks"] = clk.summary(local)
        if not per_step:
            sm_mhz = (line.get("clocks") or {}).get("sm_mhz") or 1965.0
            line["roofline"]["latency"] = latency_roofline(n, B, kms, sm_mhz, ncu_rec, tpath)
        if world == 1 and not args.no_cpu:
            v, eps_done, wall = cpu_throughput(args.workload, args.cpu_seconds, os.cpu_count(),
                                               train, args.mp_mode == "per_step")
            line["cpu_baseline"] = {
                "value": v, "unit": UNIT, "cores": os.cpu_count(), "kind": cpu_kind(),
                "sample": cpu_sample_desc(eps_done, wall, os.cpu_count(), train)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# Dependent-latency floor of one PLC decision (the chain that bounds the
# rollout kernel): dependent operations on the decision
# chain of plc_chain (fp_rollout.cuh) x their measured latencies on this B200
# (tools/micro/lat.cu, cycles per dependent trip minus its ~19-cycle loop).
# Loads from the graph tables (L1/L2) are counted as prefetchable, i.e. not
# part of the floor.
PLC_CHAIN_OPS = {          # op: (dependent count per decision, latency cycles)
    "LDS round trip (order, dev/tend, xd column, stats, xn, flag)": (6, 23),
    "fp64 add/fma (column sums 8 + centred squares 3x8 + pre-activation 8 + misc 13)": (53, 4),
    "SHFL (transpose reduction 5, device scan 3, broadcasts 3)": (11, 7),
    "REDUX (fp64 max as two 32-bit reductions) x2": (2, 20),
    "fp64 exp (device softmax)": (1, 154),
    "fp64 rsqrt (column scale, one per column since the rsqrt statistics)": (1, 64),
}


def latency_roofline(n, B, kernel_ms, sm_mhz, ncu_rec, src):
    """The rollout kernel against its latency bound: every episode of the
    batch is in flight at once (one wave up to 8 x 148 episodes), so the
    kernel time is the per-episode chain; per decision that is
    kernel_cycles / n, against the dependent-latency floor above."""
    waves = -(-B // (8 * 148))
    cycles = kernel_ms * 1e-3 * sm_mhz * 1e6 / waves
    floor = sum(c * l for c, l in PLC_CHAIN_OPS.values())
    out = {"unit": "cycles per decision", "achieved": cycles / n, "floor": floor,
           "frac": floor / (cycles / n), "waves": waves,
           "floor_model": "PLC decision chain: dependent op counts x tools/micro/lat.cu latencies "
                          "(bench.PLC_CHAIN_OPS, DESIGN.md section 4)"}
    if ncu_rec:
        inst = ncu_rec["inst_executed"]
        out["warp_instructions_per_decision"] = inst / (B * n)
        out["ipc_per_sm"] = ncu_rec.get("ipc")
        out["ncu_source"] = str(src.relative_to(ROOT))
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    procs = os.cpu_count() or 1
    total_eps = 0
    wall = 0.0
    for _ in range(args.warmup):
        cpu_throughput(args.workload, 1.0, procs, args.mode == "train",
                       args.mp_mode == "per_step")
    for _ in range(args.steps):
        v, e, w = cpu_throughput(args.workload, args.ref_step_seconds, procs,
                                 args.mode == "train", args.mp_mode == "per_step")
        total_eps += e
        wall += w
    value = total_eps / wall
    _, _, desc = workload(args.workload)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 0, "impl": "reference",
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (builder graph; random-init policy seed 0)",
        "config": bench_config(args, world, desc),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": cpu_kind(),
                         "sample": cpu_sample_desc(total_eps, wall, procs, args.mode == "train") +
                         f"; {args.steps} steps of {args.ref_step_seconds}s"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="llama_block")
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--mode", default="rollout", choices=("rollout", "train"))
    ap.add_argument("--mp-mode", default="per_episode", choices=("per_episode", "per_step"),
                    help="message passing once per snapshot (reference default) or per step")
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--encoder", default="dmma", choices=("dmma", "tc"),
                    help="GNN node MLPs: fp64 DMMA (reference-exact) or bf16 tcgen05")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-step-seconds", type=float, default=4.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--full-outputs", action="store_true",
                    help="also produce the per-step trace (log-probs, entropies, argmax) the "
                         "reference rollout returns: the general, non-lean kernel")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
