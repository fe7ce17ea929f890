"""GPU: the reference-side drop-in actually exercised.  The reference
(``flowplace``, built into oracle/_ref by oracle/build_ref.sh) is copied, the
``cuda`` backend installed exactly as INTEGRATION.md describes
(integration/install_cuda_backend.py: ``_cudacore.py`` binding
``fp_run_packed`` + the two-line dispatch in simulate.py), and the reference's
own backend-parity pattern runs against it on every golden simulator case."""
import json
import os
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "oracle" / "_ref"

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not (REF / "flowplace" / "simulate.py").exists(),
                                 reason="oracle/_ref not built (oracle/build_ref.sh)")]


def test_reference_with_cuda_backend_matches_its_python_core(tmp_path):
    sys.path.insert(0, str(ROOT))
    from integration.install_cuda_backend import install
    shutil.copytree(REF / "flowplace", tmp_path / "flowplace")
    install(tmp_path)
    env = dict(os.environ, PYTHONPATH=str(tmp_path))
    env.pop("FLOWPLACE_SIM_BACKEND", None)
    out = subprocess.run([sys.executable, str(ROOT / "tests" / "refshim_check.py"),
                          str(ROOT / "tests" / "golden" / "sim_cases.json")],
                         capture_output=True, text=True, env=env, timeout=600, cwd=tmp_path)
    assert out.returncode == 0, out.stderr[-3000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["cases"] >= 181 and res["deadlock_cases"] >= 1
    assert res["cudacore"].startswith(str(tmp_path))
