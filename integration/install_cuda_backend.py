"""Install the B200 simulator core as a ``FLOWPLACE_SIM_BACKEND=cuda`` backend
into a flowplace package tree (the edit a reference maintainer would make,
INTEGRATION.md section 1):

    python integration/install_cuda_backend.py <dir containing flowplace/> [lib.so]

1. copies ``_cudacore.py`` (the ctypes binding of ``fp_run_packed``) into
   ``flowplace/`` with the library path filled in;
2. ``simulate.backend_name`` (simulate.py:41-49) accepts ``cuda``;
3. ``simulate.exec_time`` (simulate.py:262-265) dispatches ``cuda`` to
   ``_cudacore.run_packed`` -- the same packed arguments the Cython core gets.

Idempotent.  Nothing else in the reference changes."""

from __future__ import annotations

import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
DEFAULT_LIB = HERE.parent / "paper_2505_23131_b200" / "_flowplace_b200.so"

_SEL_OLD = '''    forced = os.environ.get("FLOWPLACE_SIM_BACKEND", "auto")
'''
_SEL_NEW = '''    forced = os.environ.get("FLOWPLACE_SIM_BACKEND", "auto")
    if forced == "cuda":
        return "cuda"
'''
_RUN_OLD = '''    if backend_name() == "cython":
        makespan, raw = _simcore.run_packed(*packed)
'''
_RUN_NEW = '''    backend = backend_name()
    if backend == "cuda":
        from . import _cudacore
        makespan, raw = _cudacore.run_packed(*packed)
    elif backend == "cython":
        makespan, raw = _simcore.run_packed(*packed)
'''


def install(tree: Path, lib: Path = DEFAULT_LIB) -> Path:
    pkg = Path(tree) / "flowplace"
    sim = pkg / "simulate.py"
    src = sim.read_text()
    if "_cudacore" not in src:
        for old, new in ((_SEL_OLD, _SEL_NEW), (_RUN_OLD, _RUN_NEW)):
            if src.count(old) != 1:
                raise RuntimeError(f"{sim}: anchor not found:\n{old}")
            src = src.replace(old, new)
        sim.write_text(src)
    core = (HERE / "_cudacore.py").read_text().replace("@FLOWPLACE_B200_LIB@",
                                                       str(Path(lib).resolve()))
    (pkg / "_cudacore.py").write_text(core)
    return pkg


if __name__ == "__main__":
    tree = Path(sys.argv[1])
    lib = Path(sys.argv[2]) if len(sys.argv) > 2 else DEFAULT_LIB
    print(install(tree, lib))
