"""ctypes binding of the C ABI in include/nsnkv_b200.h.

The shared library is the product; there is no CPU fallback.  Importing this
module loads ``libnsnkv_b200.so`` from the package directory (building it
with nvcc first when it is missing and nvcc is available) and raises
ImportError when that is impossible, so a GPU box without the extension fails
loudly instead of silently running something else.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import raise_for_status

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["NSNKV_LIB"]) if os.environ.get("NSNKV_LIB") else _PKG / "libnsnkv_b200.so"


def _load() -> ctypes.CDLL:
    if not LIB_PATH.exists() or os.environ.get("NSNKV_REBUILD") == "1":
        try:
            from .build import build

            build(force=os.environ.get("NSNKV_REBUILD") == "1")
        except Exception as e:  # pragma: no cover - depends on toolchain
            raise ImportError(f"libnsnkv_b200.so is missing and could not be built: {e}") from e
    return ctypes.CDLL(str(LIB_PATH))


lib = _load()

c_void_p = ctypes.c_void_p
c_int = ctypes.c_int32
c_i64 = ctypes.c_int64
c_size = ctypes.c_size_t
c_double = ctypes.c_double


class CacheView(ctypes.Structure):
    """Mirror of struct nsnkv_cache_view."""

    _fields_ = [
        ("k_pool", c_void_p),
        ("v_pool", c_void_p),
        ("page_table", c_void_p),
        ("page_table_stride", c_int),
        ("n_chunks", c_void_p),
        ("k_res", c_void_p),
        ("v_res", c_void_p),
        ("n_res", c_void_p),
        ("base_pos", c_void_p),
        ("batch", c_int),
        ("n_kv_heads", c_int),
        ("n_q_heads", c_int),
        ("max_tokens", c_int),
        ("rope_cs", c_void_p),
        ("rope_pos0", c_i64),
        ("rope_n", c_i64),
        ("cb_k", c_void_p),
        ("cb_v", c_void_p),
        ("total_chunks", c_i64),
        ("precision", c_int),
    ]


class AppendArgs(ctypes.Structure):
    """Mirror of struct nsnkv_append_args."""

    _fields_ = [
        ("n_units", c_int),
        ("max_flush", c_int),
        ("fresh_k", c_void_p),
        ("fresh_v", c_void_p),
        ("fresh_bf16", c_int),
        ("n_new_uniform", c_i64),
        ("new_count", c_void_p),
        ("fresh_off", c_void_p),
        ("fresh_row_stride", c_i64),
        ("k_res", c_void_p),
        ("v_res", c_void_p),
        ("n_chunks_in", c_void_p),
        ("n_res_in", c_void_p),
        ("n_chunks_out", c_void_p),
        ("n_res_out", c_void_p),
        ("base_pos", c_void_p),
        ("page_table", c_void_p),
        ("page_table_stride", c_int),
        ("new_pages", c_void_p),
        ("k_pool", c_void_p),
        ("v_pool", c_void_p),
        ("counters", c_void_p),
        ("rope_cs", c_void_p),
        ("rope_pos0", c_i64),
        ("rope_n", c_i64),
        ("cb_k", c_void_p),
        ("cb_v", c_void_p),
        ("strategy", c_int),
    ]


_SIGS = {
    "nsnkv_version": ([], c_int),
    "nsnkv_last_error": ([], ctypes.c_char_p),
    "nsnkv_launch_count": ([], c_i64),
    "nsnkv_fwht_rows": ([c_void_p, c_void_p, c_i64, c_int, c_void_p], c_int),
    "nsnkv_match_block": ([c_void_p, c_i64, c_void_p, c_void_p, c_int, c_void_p, c_void_p,
                           c_void_p, c_void_p, c_void_p], c_int),
    "nsnkv_codebook_create": ([c_void_p, c_void_p, c_int, ctypes.POINTER(c_void_p)], c_int),
    "nsnkv_codebook_destroy": ([c_void_p], c_int),
    "nsnkv_codebook_bit_mode": ([c_void_p], c_int),
    "nsnkv_rope_table": ([c_void_p, c_i64, c_i64, c_void_p, c_void_p], c_int),
    "nsnkv_encode_chunks": ([c_void_p, c_int, c_void_p, c_int, c_i64, c_int, c_int, c_int,
                             c_void_p, c_void_p, c_i64, c_i64, c_void_p, c_int, c_void_p,
                             c_void_p, c_int, c_void_p, c_void_p], c_int),
    "nsnkv_decode_scores": ([ctypes.POINTER(CacheView), c_void_p, c_void_p, c_void_p], c_int),
    "nsnkv_decode_output": ([ctypes.POINTER(CacheView), c_void_p, c_void_p, c_void_p, c_size,
                             c_void_p], c_int),
    "nsnkv_decode_attend": ([ctypes.POINTER(CacheView), c_void_p, c_void_p, c_void_p, c_void_p,
                             c_size, c_void_p], c_int),
    "nsnkv_decode_workspace_bytes": ([ctypes.POINTER(CacheView)], c_size),
    "nsnkv_append": ([ctypes.POINTER(AppendArgs), c_void_p], c_int),
    "nsnkv_kmeans_assign": ([c_void_p, c_i64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                             c_void_p], c_int),
    "nsnkv_finetune_stats": ([c_void_p, c_i64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                              c_void_p, c_void_p], c_int),
    "nsnkv_decode_step": ([ctypes.POINTER(CacheView), c_void_p, c_void_p, c_void_p, c_int, c_int,
                           c_void_p, c_void_p, c_void_p, c_void_p, c_size, c_void_p], c_int),
    "nsnkv_pool_create": ([c_size, ctypes.POINTER(c_void_p)], c_int),
    "nsnkv_pool_reserve": ([c_void_p, c_size], c_int),
    "nsnkv_pool_ptr": ([c_void_p], c_void_p),
    "nsnkv_pool_mapped": ([c_void_p], c_size),
    "nsnkv_pool_destroy": ([c_void_p], c_int),
    "nsnkv_pages_copy": ([c_void_p, c_int, c_void_p, c_int, c_void_p, c_int, c_void_p], c_int),
}

EXPORTED = tuple(_SIGS)

_missing = [n for n in _SIGS if not hasattr(lib, n)]
if _missing:
    raise ImportError(f"{LIB_PATH} is stale (missing {', '.join(_missing)}); rebuild it with "
                      f"python {_PKG / 'build.py'}")

for _name, (_args, _res) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.argtypes = _args
    _fn.restype = _res


def check(code: int) -> None:
    """Raise the package exception matching a C status code."""
    if code != 0:
        msg = lib.nsnkv_last_error()
        raise_for_status(code, msg.decode() if msg else "")


def launch_count() -> int:
    return int(lib.nsnkv_launch_count())
