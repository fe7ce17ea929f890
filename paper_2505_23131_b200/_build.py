"""Compile the CUDA library in-tree for sm_100a (no JIT cache: the built .so
travels with the repo snapshot to the GPU box).

    python -m paper_2505_23131_b200._build [--force]
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
ROOT = PKG.parent
LIB = PKG / "_flowplace_b200.so"
PROF_LIB = PKG / "_flowplace_b200_prof.so"  # phase-profiling build (tools/ only)
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def deps() -> list[Path]:
    return sources() + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "flowplace_b200.h"]


def stale(lib: Path = LIB) -> bool:
    if not lib.exists():
        return True
    t = lib.stat().st_mtime
    return any(p.stat().st_mtime > t for p in deps())


def build(force: bool = False, verbose: bool = False, profile: bool = False) -> Path:
    lib = PROF_LIB if profile else LIB
    if not force and not stale(lib):
        return lib
    # objects outside the tree: only the linked .so travels to the GPU box
    import tempfile
    objdir = Path(tempfile.gettempdir()) / ("fp_b200_build_prof" if profile else "fp_b200_build")
    objdir.mkdir(exist_ok=True)
    objs = []
    flags = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                    "--expt-relaxed-constexpr", "-I", str(ROOT / "include")]
    if verbose:
        flags += ["-Xptxas", "-v"]
    if profile:
        flags += ["-DFP_PHASE_PROFILE", "-DFP_SMALL_TIMING"]
    # one nvcc per translation unit, all in parallel
    procs = []
    for src in sources():
        obj = objdir / (src.stem + ".o")
        cmd = [nvcc(), "-c", str(src), "-o", str(obj)] + flags
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                            text=True)))
        objs.append(str(obj))
    failed = []
    for src, pr in procs:
        _, err = pr.communicate()
        if pr.returncode != 0:
            failed.append(f"nvcc failed for {src.name}:\n{err}")
        elif verbose and err:
            print(err, file=sys.stderr)
    if failed:
        raise RuntimeError("\n".join(failed))
    tmp = lib.with_suffix(".so.tmp")
    cmd = [nvcc(), "-shared", "-o", str(tmp)] + [str(o) for o in objs] + ARCH + [
        "-Xcompiler", "-fPIC"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{r.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv,
                profile="--profile" in sys.argv))
