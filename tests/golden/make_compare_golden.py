"""Golden vectors for the compare evaluation (reference cli.py:316-366
``cmd_compare``'s evaluate loop: one clean exec_time at seed 0 and ``trials``
jittered ones at seeds seed + t per assignment; metrics.py pearson /
spearman), dumped from the REFERENCE in the build container:

    python tests/golden/make_compare_golden.py [--ref /root/reference/pkg]

Writes tests/golden/compare_cases.json: per case the graph (builder args),
cluster, the assignments (single, random_assign seeds, probes) with the
reference's per-row clean / noisy statistics and correlations, plus metric
known answers with ties.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))

from make_golden import _ref_imports  # noqa: E402


def compare_cases():
    import numpy as np
    from flowplace import builders
    from flowplace.cluster import ClusterSpec
    from flowplace.heuristics import random_assign, single_device_assign
    from flowplace.metrics import pearson, spearman
    from flowplace.simulate import exec_time

    cases = []
    for tag, g, cl, trials, sigma, seed, strategy in (
            ("ffnn64_d8", builders.build_ffnn(8, 4, 16, 4, 2),
             ClusterSpec.uniform(8, rate=1e6, bandwidth=1e5), 6, 0.1, 3, "fifo"),
            ("chainmm_d4_df", builders.build_chainmm(64, 2),
             ClusterSpec.uniform(4, rate=1e6, bandwidth=1e5), 4, 0.25, 11, "depth_first")):
        jittered = ClusterSpec.from_dict({**cl.to_dict(), "jitter_sigma": sigma})
        pairs = [("single", single_device_assign(g)),
                 ("random", random_assign(g, cl.device_count, seed=seed))]
        pairs += [(f"probe_{k}", random_assign(g, cl.device_count, seed=seed + 1000 + k))
                  for k in range(3)]
        rows, cs, ns = [], [], []
        for name, a in pairs:
            clean, _ = exec_time(g, a, cl, strategy, seed=0)
            noisy = [exec_time(g, a, jittered, strategy, seed=seed + t)[0] for t in range(trials)]
            rows.append({"engine": name, "clean_ms": clean,
                         "noisy_mean_ms": float(np.mean(noisy)),
                         "noisy_std_ms": float(np.std(noisy)),
                         "assignment": [int(x) for x in a]})
            cs.append(clean)
            ns.append(float(np.mean(noisy)))
        cases.append({"tag": tag, "builder": tag.split("_")[0], "devices": cl.device_count,
                      "trials": trials, "jitter_sigma": sigma, "seed": seed,
                      "strategy": strategy, "rows": rows,
                      "pearson": pearson(cs, ns), "spearman": spearman(cs, ns)})
    metrics = []
    for x, y in (([1.0, 2.0, 3.0, 4.0], [2.0, 1.0, 4.0, 3.0]),
                 ([1.0, 1.0, 2.0, 3.0, 3.0, 3.0], [6.0, 5.0, 4.0, 4.0, 2.0, 1.0]),
                 ([0.5, 0.25, 0.25, 7.0], [3.0, 3.0, 3.0, 4.0])):
        metrics.append({"x": x, "y": y, "pearson": pearson(x, y), "spearman": spearman(x, y)})
    return {"cases": cases, "metrics": metrics}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg")
    args = ap.parse_args()
    _ref_imports(Path(args.ref))
    out = HERE / "compare_cases.json"
    out.write_text(json.dumps(compare_cases(), indent=1))
    print(out)


if __name__ == "__main__":
    main()
