"""Level-1 drop-in: the reference kernel plug-in backed by sm_100a CUDA.

Same module surface as reference pkg/src/nsnkv/kernels/__init__.py:25-59
(``fwht_rows``, ``match_block``, ``entry_inv_norms``, ``backends``,
``BACKEND``), so it can be registered next to the reference's ``native`` and
``python`` backends and run through the reference's own bit-parity tests
(pkg/tests/test_kernels_parity.py).  Host numpy arrays in, host numpy arrays
out, exactly the reference signatures; device-tensor variants
(``fwht_rows_t``, ``match_block_t``) skip the copies.

There is no CPU path: every call runs the CUDA kernels of libnsnkv_b200.so.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .codebook import entry_inv_norms  # noqa: F401  (re-export, reference parity)

BACKEND = "cuda"
HAVE_NATIVE = True


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("the nsnkv CUDA backend needs a CUDA device")
    return torch.device("cuda", torch.cuda.current_device())


def fwht_rows_t(a: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """Orthonormal FWHT of each row of a CUDA fp32 [n, d] tensor."""
    if a.dtype != torch.float32 or a.dim() != 2 or not a.is_cuda:
        raise ValueError("fwht_rows_t expects a 2-D CUDA float32 tensor")
    a = a.contiguous()
    out = torch.empty_like(a) if out is None else out
    _lib.check(_lib.lib.nsnkv_fwht_rows(a.data_ptr(), out.data_ptr(), a.shape[0], a.shape[1],
                                        _stream()))
    return out


def fwht_rows(a: np.ndarray) -> np.ndarray:
    """Reference signature (_native.pyx:16): new fp32 array, input untouched."""
    x = np.ascontiguousarray(a, dtype=np.float32)
    if x.ndim != 2:
        raise ValueError("fwht_rows expects a 2-D array")
    if x.shape[0] == 0:
        return x.copy()
    t = torch.from_numpy(x).to(_device())
    return fwht_rows_t(t).cpu().numpy()


def match_block_t(vecs: torch.Tensor, entries: torch.Tensor, inv_norms: torch.Tensor, fold: bool,
                  want_zero_mask: bool = False, neartie: torch.Tensor | None = None):
    """Device variant: returns (idx u8, signs u8 | None, zero_mask u8 | None)."""
    m = vecs.shape[0]
    dev = vecs.device
    idx = torch.empty(m, dtype=torch.uint8, device=dev)
    signs = torch.empty(m, dtype=torch.uint8, device=dev) if fold else None
    zm = torch.empty(m, dtype=torch.uint8, device=dev) if want_zero_mask else None
    _lib.check(_lib.lib.nsnkv_match_block(
        vecs.contiguous().data_ptr(), m, entries.contiguous().data_ptr(),
        inv_norms.contiguous().data_ptr(), 1 if fold else 0, idx.data_ptr(),
        signs.data_ptr() if signs is not None else None,
        zm.data_ptr() if zm is not None else None,
        neartie.data_ptr() if neartie is not None else None, _stream()))
    return idx, signs, zm


def match_block(vecs, entries, inv_norms, fold):
    """Reference signature (kernels/__init__.py:35-41 and _native.pyx:41-87):
    (idx u8[m], signs u8[m] | None).  Like the reference kernel this does not
    substitute zero rows; codebook-level callers do (see match_rows)."""
    v = np.ascontiguousarray(vecs, dtype=np.float32)
    e = np.ascontiguousarray(entries, dtype=np.float32)
    inv = np.ascontiguousarray(inv_norms, dtype=np.float64)
    if v.ndim != 2 or v.shape[1] != 8:
        raise ValueError(f"expected (m, 8) sub-vectors, got {v.shape}")
    if v.shape[0] == 0:
        return np.empty(0, np.uint8), (np.empty(0, np.uint8) if fold else None)
    dev = _device()
    idx, signs, _ = match_block_t(torch.from_numpy(v).to(dev), torch.from_numpy(e).to(dev),
                                  torch.from_numpy(inv).to(dev), bool(fold))
    return idx.cpu().numpy(), (signs.cpu().numpy() if fold else None)


def match_rows(vecs, entries, inv_norms, fold):
    """codebook.match_block semantics (codebook.py:109-128): returns
    (idx, signs | None, zero_mask bool) with zero rows substituted."""
    v = np.ascontiguousarray(vecs, dtype=np.float32)
    if v.shape[0] == 0:
        z = np.empty(0, np.uint8)
        return z, (z.copy() if fold else None), np.zeros(0, bool)
    dev = _device()
    idx, signs, zm = match_block_t(
        torch.from_numpy(v).to(dev),
        torch.from_numpy(np.ascontiguousarray(entries, dtype=np.float32)).to(dev),
        torch.from_numpy(np.ascontiguousarray(inv_norms, dtype=np.float64)).to(dev),
        bool(fold), want_zero_mask=True)
    return (idx.cpu().numpy(), signs.cpu().numpy() if signs is not None else None,
            zm.cpu().numpy().astype(bool))


def backends() -> dict:
    """Backends this module provides (reference kernels/__init__.py:54-59)."""
    import sys

    return {"cuda": sys.modules[__name__]}
