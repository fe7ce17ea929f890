"""bench.py's JSON-line contract (the driver parses it): the reference arm on
CPU, our arm on the GPU."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _run(args, timeout):
    env = dict(os.environ, PYTHONPATH=str(ROOT))
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True,
                         text=True, timeout=timeout, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "3", "--ref-step-seconds", "0.5"],
             timeout=300)
    assert d["impl"] == "reference"
    assert d["metric"] == "simulated placement episodes/sec" and d["unit"] == "episodes/s"
    assert d["value"] > 0 and d["higher_is_better"] is True
    ref_built = (ROOT / "oracle" / "_ref" / "flowplace" / "policy.py").exists()
    assert d["cpu_baseline"]["kind"] == ("reference" if ref_built else "port")
    assert d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("Llama-7B block")
    assert d["config"]["episodes_per_gpu"] == 1024 and d["config"]["global_batch"] == 1024


@pytest.mark.gpu
def test_our_arm_line():
    d = _run(["--steps", "2", "--warmup", "3", "--no-cpu"], timeout=600)
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
                "gpu_launches", "roofline", "clocks", "rates"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3 and d["dtype"] == "f64"
    assert d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= 2 * d["steps"]
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-12
    assert d["rates"]["decisions_per_s"] == pytest.approx(d["value"] * 208)
