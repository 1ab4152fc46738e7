"""Build the sm_100a shared library libnsnkv_b200.so in-tree with nvcc.

The library is the product: a C ABI (include/nsnkv_b200.h) over hand-written
CUDA kernels.  It is built in place so the .so travels with the repository
snapshot to the GPU box.  Usage: ``python -m paper_2505_18231_b200.build``.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libnsnkv_b200.so"

SOURCES = ["capi.cu", "level1.cu", "encode.cu", "decode_ref.cu", "decode_attend.cu", "decode_attend3.cu"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
    "--shared",
    # parity-critical arithmetic is written with explicit _rn intrinsics; keep
    # IEEE division/sqrt and denormals everywhere else as well
    "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
    "-Xptxas", "-warn-spills",
]


def nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def needs_rebuild() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "nsnkv_b200.h"]
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False, trace: bool = False) -> Path:
    """trace=True builds libnsnkv_b200_trace.so with -DNSNKV_TRACE (a debug
    timeline of CTA 0 in the decode kernel, scripts/trace_decode.py).
    NSNKV_EXTRA_FLAGS / NSNKV_LIB_NAME build experiment variants next to it."""
    extra = os.environ.get("NSNKV_EXTRA_FLAGS", "").split()
    lib = LIB.with_name("libnsnkv_b200_trace.so") if trace else LIB
    if extra:
        lib = lib.with_name(os.environ.get("NSNKV_LIB_NAME", lib.name))
    if not force and not trace and not extra and not needs_rebuild():
        return LIB
    cmd = [nvcc(), *NVCC_FLAGS, *(["-DNSNKV_TRACE"] if trace else []), *extra, "-I", str(ROOT / "include"),
           *[str(CSRC / s) for s in SOURCES], "-o", str(lib) + ".tmp", "-lcudart"]
    if verbose:
        print(" ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libnsnkv_b200.so")
    if verbose and (res.stdout or res.stderr):
        sys.stderr.write(res.stdout + res.stderr)
    os.replace(str(lib) + ".tmp", lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, trace="--trace" in sys.argv))
