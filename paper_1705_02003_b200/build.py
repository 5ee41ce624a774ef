"""Build libuqg.so in-tree with nvcc for sm_100a (used by __graft_entry__.build)."""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libuqg.so"
SOURCES = ["uqg_abi.cu", "uqg_kernels.cu", "uqg_pcg.cu", "uqg_persistent.cu", "uqg_surrogate.cu"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--fmad=false",           # numpy never contracts a*b+c; explicit __fma_rn where wanted
    "-Xptxas", "-v",
    "-Xcompiler", "-fPIC,-O2",
    "-cudart", "static",
    "-shared",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or Path(cand).exists()):
            return cand
    raise RuntimeError("nvcc not found")


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "uqg.h"]
    return any(p.stat().st_mtime > t for p in deps if p.exists())


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile libuqg.so.  Safe under concurrent callers (e.g. every rank of a
    torchrun job finding a stale library): one builds under an exclusive file
    lock, the others wait and reuse its result."""
    import fcntl

    if not force and not needs_build():
        return LIB
    with open(PKG / ".build.lock", "w") as lock:
        fcntl.flock(lock, fcntl.LOCK_EX)
        try:
            if not force and not needs_build():  # built by another process meanwhile
                return LIB
            tmp = f"{LIB}.tmp.{os.getpid()}"
            extra = os.environ.get("UQG_NVCC_EXTRA", "").split()  # tuning experiments
            cmd = [_nvcc(), *NVCC_FLAGS, *extra, "-I", str(PKG.parent / "include"), "-o", tmp,
                   *[str(CSRC / s) for s in SOURCES]]
            res = subprocess.run(cmd, capture_output=True, text=True)
            if verbose or res.returncode:
                sys.stderr.write(res.stdout + res.stderr)
            if res.returncode:
                raise RuntimeError(f"nvcc failed ({res.returncode})")
            os.replace(tmp, LIB)
            (PKG / "ptxas.log").write_text(res.stderr)
        finally:
            fcntl.flock(lock, fcntl.LOCK_UN)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
