"""Per-call latency of the reference's simulator FFI boundary, Cython core vs
the B200 core behind the same call (integration/_cudacore.py ->
fp_run_packed), on the GPU box:

    python tools/ref_abi_latency.py [--out gpurun_out/r2_ref_abi_latency.jsonl]

For each graph: the reference's own ``_pack`` output for a fresh random
assignment per call, then ``run_packed(*packed)`` through each core (the
exact FFI call of simulate.py:262-265), median over calls; and the whole
``exec_time`` (pack + core + _assemble) per backend.  Results must be equal
call for call."""
from __future__ import annotations

import argparse
import json
import os
import shutil
import statistics
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "r2_ref_abi_latency.jsonl"))
    ap.add_argument("--calls", type=int, default=60)
    args = ap.parse_args()
    from integration.install_cuda_backend import install
    tmp = Path(tempfile.mkdtemp())
    shutil.copytree(ROOT / "oracle" / "_ref" / "flowplace", tmp / "flowplace")
    install(tmp)
    sys.path.insert(0, str(tmp))
    import numpy as np
    from flowplace import _cudacore, _simcore, graph as G
    from flowplace import simulate as S
    from flowplace.cluster import ClusterSpec
    from flowplace.features import static_features
    from paper_2505_23131_b200 import builders
    from paper_2505_23131_b200.graph import graph_to_dict

    work = [("ffnn", builders.build_ffnn(8, 4, 16, 4, 2), ClusterSpec.uniform(8, 1e6, 1e5)),
            ("llama_block", builders.build_llama_block(), ClusterSpec.uniform(8, 1e9, 1e7)),
            ("dag1k", builders.sparse_dag(1000, seed=0), ClusterSpec.uniform(8, 1e9, 1e7)),
            ("dag10k", builders.sparse_dag(10_000, seed=0), ClusterSpec.uniform(8, 1e9, 1e7))]
    rows = []
    for name, g0, cl in work:
        g = G.graph_from_dict(graph_to_dict(g0))
        feats = static_features(g, cl.comm_factor)
        rng = np.random.default_rng(0)
        calls = args.calls if len(g) < 5000 else 8
        assigns = [[int(x) for x in rng.integers(0, cl.device_count, size=len(g))]
                   for _ in range(calls + 2)]
        packs = [S._pack(g, a, cl, feats, "fifo", 0) for a in assigns]
        res = {}
        for core_name, core in (("cython", _simcore), ("cuda", _cudacore)):
            core.run_packed(*packs[0])  # warm (cuda: builds the cached problem)
            ts, out = [], []
            for pk in packs[1:]:
                t0 = time.perf_counter()
                mk, ev = core.run_packed(*pk)
                ts.append(time.perf_counter() - t0)
                out.append((mk, ev))
            res[core_name] = (statistics.median(ts), out)
            et = []
            for backend in (core_name,):
                os.environ["FLOWPLACE_SIM_BACKEND"] = backend
                for a in assigns[1:]:
                    t0 = time.perf_counter()
                    S.exec_time(g, a, cl, "fifo", 0, feats)
                    et.append(time.perf_counter() - t0)
            res[core_name + "_exec_time"] = statistics.median(et)
        assert res["cython"][1] == res["cuda"][1], name
        row = {"graph": name, "n": len(g), "calls": calls,
               "run_packed_ms": {"cython": res["cython"][0] * 1e3, "cuda": res["cuda"][0] * 1e3},
               "exec_time_ms": {"cython": res["cython_exec_time"] * 1e3,
                                "cuda": res["cuda_exec_time"] * 1e3},
               "identical_results": True}
        row["run_packed_speedup"] = row["run_packed_ms"]["cython"] / row["run_packed_ms"]["cuda"]
        print(json.dumps(row), flush=True)
        rows.append(row)
    Path(args.out).parent.mkdir(exist_ok=True)
    Path(args.out).write_text("".join(json.dumps(r) + "\n" for r in rows))


if __name__ == "__main__":
    main()
