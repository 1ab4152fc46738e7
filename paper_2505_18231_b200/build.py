"""Build the sm_100a shared library libnsnkv_b200.so in-tree with nvcc.

The library is the product: a C ABI (include/nsnkv_b200.h) over hand-written
CUDA kernels.  It is built in place so the .so travels with the repository
snapshot to the GPU box.  Usage: ``python paper_2505_18231_b200/build.py``
(not ``-m``: importing the package loads the library it is about to rebuild).
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

SOURCES = ["capi.cu", "pool.cu", "level1.cu", "encode.cu", "decode_ref.cu", "decode_dispatch.cu", "decode_attend3.cu", "codebook_build.cu"]

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


def _deps() -> list[Path]:
    return list(CSRC.glob("*.cuh")) + [ROOT / "include" / "nsnkv_b200.h"]


def needs_rebuild() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in list(CSRC.glob("*.cu")) + _deps())


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile every translation unit to an object under build/ (in parallel,
    only the stale ones unless force), then link libnsnkv_b200.so.
    NSNKV_EXTRA_FLAGS / NSNKV_LIB_NAME build experiment variants next to it."""
    from concurrent.futures import ThreadPoolExecutor

    extra = os.environ.get("NSNKV_EXTRA_FLAGS", "").split()
    lib = LIB.with_name(os.environ.get("NSNKV_LIB_NAME", LIB.name)) if extra else LIB
    if not force and not extra and not needs_rebuild():
        return LIB
    objdir = ROOT / "build" / ("obj_" + lib.stem)
    objdir.mkdir(parents=True, exist_ok=True)
    dep_t = max(p.stat().st_mtime for p in _deps())
    flags = [f for f in NVCC_FLAGS if f != "--shared"]

    def compile_one(src: str):
        obj = objdir / (src + ".o")
        s = CSRC / src
        if not force and obj.exists() and obj.stat().st_mtime > max(s.stat().st_mtime, dep_t):
            return src, None
        cmd = [nvcc(), *flags, *extra, "-I", str(ROOT / "include"), "-c", str(s), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), flush=True)
        return src, subprocess.run(cmd, capture_output=True, text=True)

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    for src, res in results:
        if res is None:
            continue
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError(f"nvcc failed compiling {src}")
        if verbose and (res.stdout or res.stderr):
            sys.stderr.write(res.stdout + res.stderr)
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "--shared",
           *[str(objdir / (s + ".o")) for s in SOURCES], "-o", str(lib) + ".tmp", "-lcudart"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed linking libnsnkv_b200.so")
    os.replace(str(lib) + ".tmp", lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
