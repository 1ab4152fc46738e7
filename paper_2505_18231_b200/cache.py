"""Batched packed KV cache on the GPU, behind the reference pipeline API.

Reference (pkg/src/nsnkv):
  * ``CacheConfig``            kvcache.py:33-45
  * ``ScaleStrategy``          vq.py:31-48
  * residual policy / append   kvcache.py:48-74, 157-195
  * flush_chunk_keys/values    kvcache.py:114-154  -> nsnkv_encode_chunks
  * scores_quantized           attention.py:83-111 -> nsnkv_decode_scores
  * output_quantized           attention.py:114-133 -> nsnkv_decode_output
  * attend_quantized           attention.py:136-142 -> nsnkv_decode_attend
  * snapshot / wire format     kvcache.py:198-213, vq.py:363-380

``PagedKvCache`` holds B x H_kv independent units (one reference
``KvCacheState`` each, with its own length) in device memory: packed pages
for every flushed 64-token chunk (K and V pools on growable virtual memory),
a free list, a page table, and the fp32 residual rows.  Appends are uniform
([B, H, n, 128]) or ragged (packed rows + per-sequence lengths), one kernel
launch each; sequences are released and imported from reference snapshots.
The single-head facade in ``api.py`` is a 1 x 1 batch.
"""

from __future__ import annotations

import ctypes
import enum
import os
import math
import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .codebook import BitMode, Codebook
from .errors import FormatError, IndexOutOfRange, ShapeMismatch, Unsupported

D = 128
R = 64
NPAIR = D // 2
PAGE_BYTES = {BitMode.TWO_BIT: 2304, BitMode.ONE_BIT: 1280}
LEDGER_BYTES = {BitMode.TWO_BIT: 2292, BitMode.ONE_BIT: 1268}
CNT_CLAMP, CNT_ZERO, CNT_FALLBACK, CNT_NEARTIE = range(4)
# decode codeword precision (C-ABI nsnkv_cache_view.precision)
PRECISIONS = {"precise": 0, "vfast": 1, "fast": 2}


def default_precision(bit_mode) -> str:
    """Key codewords always enter the score product as fp16 hi + lo: a plain
    fp16 key codeword (11-bit significand) puts a relative error of ~2^-12 on
    every score, and with large-magnitude scores (outlier tokens) that shifts
    the softmax far beyond the 1e-3 output tolerance (2-bit misaligned data,
    4K context: 3e-2).  Value codewords are plain fp16 in both
    bit modes ("vfast").  2-bit: the per-component signs make the rounding
    errors cancel (<= 2.5e-4 at 32K context).  1-bit: the unsigned codewords'
    rounding errors have a nonzero mean that would accumulate with the context
    (1.7e-3 at 4K, 4.0e-3 at 32K uncorrected); the kernel adds the codebook's
    mean rounding error times the summed weights (CodebookDev::dbar), which
    leaves 2.6e-4 at 4K and at 32K."""
    return "vfast"


def check_precision(precision: str, bit_mode, allow_inexact: bool = False) -> str:
    """Validate a precision mode for a bit mode.  "fast" (plain-fp16 key
    codewords) is known to exceed the 1e-3 output tolerance on outlier data
    and needs an explicit allow_inexact=True."""
    if precision not in PRECISIONS:
        raise ValueError(f"precision must be one of {sorted(PRECISIONS)}")
    inexact = precision == "fast"
    if inexact and not allow_inexact:
        raise Unsupported(f"precision {precision!r} exceeds the 1e-3 output tolerance on some "
                          f"{int(bit_mode)}-bit inputs; pass allow_inexact=True to use it")
    return precision


class ScaleStrategy(enum.IntEnum):
    """Reconstruction rescaling (vq.py:31-48)."""

    NONE = 0
    MIN_L2 = 1
    NORM_MATCH = 2
    PARALLEL = 3

    @staticmethod
    def parse(s) -> "ScaleStrategy":
        if isinstance(s, ScaleStrategy):
            return s
        table = {"none": ScaleStrategy.NONE, "s1": ScaleStrategy.MIN_L2,
                 "s2": ScaleStrategy.NORM_MATCH, "s3": ScaleStrategy.PARALLEL}
        key = str(s).lower()
        if key not in table:
            raise ValueError(f"unknown strategy {s!r}")
        return table[key]


@dataclass(frozen=True)
class CacheConfig:
    """Hot-path knobs (kvcache.py:33-45).  The GPU path implements d = 128,
    residual_size = 64, double quantization on, no VQ bypass; other values
    are rejected with ``Unsupported`` when a cache is created."""

    d: int
    bit_mode: BitMode
    residual_size: int = 64
    strategy: ScaleStrategy = ScaleStrategy.PARALLEL
    rope_base: float = 10000.0
    dq_enabled: bool = True
    bypass_vq: bool = False

    def __post_init__(self):
        if self.residual_size < 1:
            raise ValueError("residual_size must be >= 1")
        object.__setattr__(self, "bit_mode", BitMode.parse(self.bit_mode))
        object.__setattr__(self, "strategy", ScaleStrategy.parse(self.strategy))

    def check_gpu_path(self) -> None:
        if self.d != D:
            raise Unsupported(f"GPU path implements head_dim {D}, got {self.d}")
        if self.residual_size != R:
            raise Unsupported(f"GPU path implements residual_size {R}, got {self.residual_size}")
        if not self.dq_enabled or self.bypass_vq:
            raise Unsupported("GPU path stores double-quantized pages only (dq on, no bypass)")


# ---------------------------------------------------------------------------
# RoPE angle tables (rope.py:29-51), one per (device, base), grown on demand
# ---------------------------------------------------------------------------
def pair_freqs(d: int, base: float) -> np.ndarray:
    """base ** (-2j/d) in float64 (rope.py:29-32)."""
    j = np.arange(d // 2, dtype=np.float64)
    return float(base) ** (-2.0 * j / d)


class RopeTable:
    _tables: dict = {}

    def __init__(self, device: torch.device, base: float):
        self.device = device
        self.freqs = torch.from_numpy(pair_freqs(D, base)).to(device)
        self.cs = torch.empty(0, NPAIR, 2, dtype=torch.float32, device=device)

    @classmethod
    def get(cls, device: torch.device, base: float) -> "RopeTable":
        key = (str(device), float(base))
        t = cls._tables.get(key)
        if t is None:
            t = cls._tables[key] = RopeTable(device, base)
        return t

    def ensure(self, n_pos: int) -> torch.Tensor:
        """Table rows cover positions [0, n_pos)."""
        have = self.cs.shape[0]
        if n_pos > have:
            new_n = max(n_pos, 2 * have, 4096)
            new_n = (new_n + 63) // 64 * 64
            cs = torch.empty(new_n, NPAIR, 2, dtype=torch.float32, device=self.device)
            if have:
                cs[:have].copy_(self.cs)
            _lib.check(_lib.lib.nsnkv_rope_table(self.freqs.data_ptr(), have, new_n - have,
                                                 cs[have:].data_ptr(), _stream()))
            self.cs = cs
        return self.cs


def resolve_device(device=None) -> torch.device:
    """An indexed CUDA device: None or "cuda" without an index means the
    calling thread's current device (one process per GPU after
    torch.cuda.set_device(rank)), never GPU 0."""
    d = torch.device("cuda") if device is None else torch.device(device)
    if d.type != "cuda":
        raise Unsupported(f"the packed cache lives on a CUDA device, got {d}")
    return d if d.index is not None else torch.device("cuda", torch.cuda.current_device())


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


# ---------------------------------------------------------------------------
# the batched cache
# ---------------------------------------------------------------------------
class _Staging:
    """One pinned host staging ring per device for small uploads (page ids,
    ragged counts): a fresh pinned allocation costs ~1 ms, so the ring is
    allocated once and reused; a wrap waits for the copies still reading it."""

    _rings: dict = {}

    def __init__(self, device: torch.device, nbytes: int = 1 << 22):
        self.device = device
        self.buf = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
        self.np = self.buf.numpy()
        self.off = 0
        self.ev = torch.cuda.Event()

    @classmethod
    def get(cls, device: torch.device) -> "_Staging":
        r = cls._rings.get(str(device))
        if r is None:
            r = cls._rings[str(device)] = _Staging(device)
        return r

    def upload(self, a: np.ndarray) -> torch.Tensor:
        nb = a.nbytes
        if nb > self.buf.numel():
            return torch.from_numpy(a).to(self.device)
        off = (self.off + 255) // 256 * 256
        if off + nb > self.buf.numel():
            self.ev.synchronize()
            off = 0
        self.np[off:off + nb] = a.view(np.uint8).reshape(-1)
        out = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, device=self.device)
        out.view(-1).view(torch.uint8).copy_(self.buf[off:off + nb], non_blocking=True)
        self.ev.record()
        self.off = off + nb
        return out


class _Pool:
    """One growable page pool (C-ABI nsnkv_pool_*): a reserved virtual address
    range with physical memory mapped on demand, so growth never copies or
    moves a page."""

    def __init__(self, device: torch.device, page_bytes: int):
        self.page_bytes = page_bytes
        reserve = torch.cuda.get_device_properties(device).total_memory
        h = _lib.c_void_p()
        with torch.cuda.device(device):
            _lib.check(_lib.lib.nsnkv_pool_create(reserve, ctypes.byref(h)))
        self.handle = h.value
        self.ptr = int(_lib.lib.nsnkv_pool_ptr(self.handle))

    @property
    def pages(self) -> int:
        return int(_lib.lib.nsnkv_pool_mapped(self.handle)) // self.page_bytes

    def grow(self, pages: int) -> int:
        """Map memory for at least `pages` pages; returns the page capacity."""
        if pages > self.pages:
            _lib.check(_lib.lib.nsnkv_pool_reserve(self.handle, pages * self.page_bytes))
        return self.pages

    def __del__(self):  # pragma: no cover - interpreter shutdown order varies
        try:
            _lib.lib.nsnkv_pool_destroy(self.handle)
        except Exception:
            pass


class PagedKvCache:
    """B x H_kv units of packed KV cache on one GPU: one reference
    ``KvCacheState`` (kvcache.py:77-107) per unit, each with its own length.

    Storage: K and V page pools (one 64-token chunk of one unit per page) on
    CUDA virtual memory that grow without copying, a free list of page ids,
    a page table [units][chunks], fp32 residual rows [units][64][128] and
    per-unit chunk / residual counters on the device.  The host mirrors every
    length (it issues every append), so an append is ONE kernel launch
    (nsnkv_append: flushes, residual rows, page table and counters) with no
    device->host synchronisation; page ids for newly flushed chunks come from
    the free list and are uploaded with the launch only when a unit flushes.
    Sequences end with ``release`` (pages return to the free list) and start
    from reference snapshots with ``load_snapshot`` / ``import_unit``.
    """

    def __init__(self, config: CacheConfig, batch: int, n_kv_heads: int, max_tokens: int = 0,
                 cb_k: Codebook | None = None, cb_v: Codebook | None = None,
                 base_position: int = 0, device=None, check_finite: bool = True,
                 precision: str | None = None, allow_inexact: bool = False):
        config.check_gpu_path()
        if precision is None:  # deployment default; NSNKV_PRECISION overrides
            precision = os.environ.get("NSNKV_PRECISION") or default_precision(config.bit_mode)
        # check_finite mirrors the reference's as_tensor2d validation
        # (core.py:38); it costs one device->host sync per append, so a server
        # that validates its activations elsewhere passes False
        self.check_finite = check_finite
        self.precision = check_precision(precision, config.bit_mode, allow_inexact)
        if batch < 1 or n_kv_heads < 1:
            raise ShapeMismatch("batch and n_kv_heads must be >= 1")
        if int(base_position) < 0:
            raise Unsupported("base_position must be >= 0 (the RoPE table starts at position 0)")
        self.config = config
        self.batch = batch
        self.n_kv_heads = n_kv_heads
        self.units = batch * n_kv_heads
        self.device = resolve_device(device)
        self.bit_mode = config.bit_mode
        self.page_bytes = PAGE_BYTES[self.bit_mode]
        self.cb_k = cb_k
        self.cb_v = cb_v
        self.base_position = int(base_position)
        U, dev = self.units, self.device
        # host mirrors of the per-unit state (exact: every change goes through here)
        self.unit_n_chunks = np.zeros(U, np.int64)
        self.unit_n_res = np.zeros(U, np.int64)
        self.unit_total = np.zeros(U, np.int64)
        self.unit_base = np.full(U, self.base_position, np.int64)
        self._pt = np.zeros((U, 0), np.int32)          # page table mirror
        self._free = np.zeros(0, np.int32)              # free page ids (stack, top = end)
        # device state
        self.k_res = torch.zeros(U, R, D, dtype=torch.float32, device=dev)
        self.v_res = torch.zeros(U, R, D, dtype=torch.float32, device=dev)
        self._cnt = torch.zeros(2, 2, U, dtype=torch.int32, device=dev)  # [buf][chunks, res][unit]
        self._cur = 0
        self.base_pos_t = torch.full((U,), self.base_position, dtype=torch.int64, device=dev)
        self.page_table = torch.zeros(U, 0, dtype=torch.int32, device=dev)
        self._events = torch.zeros(0, 2, 4, dtype=torch.int32, device=dev)  # [page][K, V][counter]
        self._pools = {"k": _Pool(dev, self.page_bytes), "v": _Pool(dev, self.page_bytes)}
        self._ws = torch.empty(0, dtype=torch.uint8, device=dev)
        self._keep = []  # host buffers of in-flight uploads
        self.rope = RopeTable.get(dev, config.rope_base)
        if max_tokens:
            self.reserve(max_tokens)

    # -- storage ------------------------------------------------------------
    @property
    def capacity(self) -> int:
        """Pages mapped in each pool."""
        return self._events.shape[0]

    def _grow_pages(self, need_free: int) -> None:
        if self._free.size >= need_free:
            return
        old = self.capacity
        want = old + (need_free - self._free.size)
        want = max(want, old + old // 4, 64)
        new = min(self._pools["k"].grow(want), self._pools["v"].grow(want))
        ev = torch.zeros(new, 2, 4, dtype=torch.int32, device=self.device)
        if old:
            ev[:old].copy_(self._events)  # per-page event counters (32 B a page)
        self._events = ev
        # new ids pushed in descending order, so pops hand out ascending runs
        self._free = np.concatenate([np.arange(new - 1, old - 1, -1, dtype=np.int32), self._free])

    def _alloc(self, n: int) -> np.ndarray:
        self._grow_pages(n)
        ids = self._free[self._free.size - n:][::-1].copy()
        self._free = self._free[:self._free.size - n]
        return ids

    def _ensure_width(self, chunks: int) -> None:
        W = self._pt.shape[1]
        if chunks <= W:
            return
        new = max(chunks, 2 * W, 16)
        pt = np.zeros((self.units, new), np.int32)
        pt[:, :W] = self._pt
        self._pt = pt
        t = torch.zeros(self.units, new, dtype=torch.int32, device=self.device)
        if W:
            t[:, :W].copy_(self.page_table)
        self.page_table = t

    def reserve(self, max_tokens: int) -> "PagedKvCache":
        """Pre-size pools, page table and RoPE table so every unit can hold
        max_tokens tokens (a server reserves up front; growth later maps more
        memory without copying pages)."""
        n = (int(max_tokens) + R - 1) // R
        need = int(np.maximum(n - self.unit_n_chunks, 0).sum())
        self._grow_pages(need)
        self._ensure_width(n)
        self.rope.ensure(int(self.unit_base.max()) + n * R + R)
        return self

    def pool_ptrs(self) -> tuple[int, int]:
        return self._pools["k"].ptr, self._pools["v"].ptr

    # -- lengths -------------------------------------------------------------
    @property
    def n_chunks(self) -> int:
        """Flushed chunks (max over units; equal for uniform appends)."""
        return int(self.unit_n_chunks.max())

    @property
    def n_res(self) -> int:
        return int(self.unit_n_res.max())

    @property
    def total_tokens(self) -> int:
        return int(self.unit_total.max())

    @property
    def n_quantized(self) -> int:
        return self.n_chunks * R

    @property
    def max_chunks(self) -> int:
        return self._pt.shape[1]

    @property
    def max_tokens(self) -> int:
        """Row stride of score / weight buffers (a multiple of 64)."""
        n = self.unit_n_chunks + (self.unit_n_res > 0)
        return max(R, int(n.max()) * R)

    # -- append (kvcache.py:157-195) ------------------------------------------
    def append(self, keys, values, cb_k: Codebook | None = None,
               cb_v: Codebook | None = None, seq_lens=None) -> "PagedKvCache":
        """Append keys (pre-RoPE) and values (post-HT).

        Uniform: [B, H_kv, n, 128] (every unit gains n tokens).  Ragged
        (``seq_lens``, B ints): packed [sum(seq_lens), H_kv, 128], sequence b
        contributing rows sum(seq_lens[:b]) .. + seq_lens[b] (zero = no
        tokens this step).  One kernel launch either way."""
        cb_k = cb_k or self.cb_k
        cb_v = cb_v or self.cb_v
        if cb_k is None or cb_v is None:
            raise ShapeMismatch("append needs the key and value codebooks")
        if cb_k.bit_mode != self.bit_mode or cb_v.bit_mode != self.bit_mode:
            raise ShapeMismatch("codebook bit mode does not match the cache")
        self.cb_k, self.cb_v = cb_k, cb_v
        U = self.units
        if seq_lens is None:
            k = self._as_rows(keys)
            v = self._as_rows(values)
            if k.shape != v.shape:
                raise ShapeMismatch("key and value batches must have the same shape")
            n = k.shape[1]
            if n < 1:
                raise ShapeMismatch("append needs at least one token")
            n_new = np.full(U, n, np.int64)
            counts_t = offs_t = None
            row_stride = 1
        else:
            lens = np.asarray(seq_lens, np.int64).reshape(-1)
            if lens.shape[0] != self.batch or (lens < 0).any():
                raise ShapeMismatch(f"seq_lens must hold {self.batch} non-negative lengths")
            k = self._as_packed(keys, int(lens.sum()))
            v = self._as_packed(values, int(lens.sum()))
            if k.shape != v.shape:
                raise ShapeMismatch("key and value batches must have the same shape")
            if not lens.any():
                return self
            H = self.n_kv_heads
            cu = np.concatenate([[0], np.cumsum(lens)])
            n_new = np.repeat(lens, H)
            offs = (cu[:-1, None] * H + np.arange(H)[None, :]).reshape(-1)
            counts_t = self._upload(n_new.astype(np.int32))
            offs_t = self._upload(offs.astype(np.int64))
            n = 0
            row_stride = H
        if k.dtype != v.dtype:  # one fp32 / one bf16 batch: encode both from fp32
            k, v = k.float(), v.float()
        n_flush = (self.unit_n_res + n_new) // R
        fmax = int(n_flush.max())
        new_pages_t = None
        if fmax:
            self._ensure_width(int((self.unit_n_chunks + n_flush).max()))
            ids = self._alloc(int(n_flush.sum()))
            # unit-major: unit u takes the next n_flush[u] ids
            mask = np.arange(fmax)[None, :] < n_flush[:, None]
            npg = np.zeros((U, fmax), np.int32)
            npg[mask] = ids
            rows, ks = np.nonzero(mask)
            self._pt[rows, self.unit_n_chunks[rows] + ks] = ids
            new_pages_t = self._upload(npg)
        table = self.rope.ensure(int((self.unit_base + (self.unit_n_chunks + n_flush) * R).max()) + R)
        a = _lib.AppendArgs()
        a.n_units, a.max_flush = U, fmax
        a.fresh_k, a.fresh_v = k.data_ptr(), v.data_ptr()
        a.fresh_bf16 = 1 if k.dtype == torch.bfloat16 else 0
        a.n_new_uniform = n
        a.new_count = counts_t.data_ptr() if counts_t is not None else None
        a.fresh_off = offs_t.data_ptr() if offs_t is not None else None
        a.fresh_row_stride = row_stride
        a.k_res, a.v_res = self.k_res.data_ptr(), self.v_res.data_ptr()
        src, dst = self._cnt[self._cur], self._cnt[1 - self._cur]
        a.n_chunks_in, a.n_res_in = src[0].data_ptr(), src[1].data_ptr()
        a.n_chunks_out, a.n_res_out = dst[0].data_ptr(), dst[1].data_ptr()
        a.base_pos = self.base_pos_t.data_ptr()
        a.page_table = self.page_table.data_ptr() if self.page_table.numel() else None
        a.page_table_stride = self.page_table.stride(0) if self.page_table.numel() else 0
        a.new_pages = new_pages_t.data_ptr() if new_pages_t is not None else None
        a.k_pool, a.v_pool = self.pool_ptrs()
        a.counters = self._events.data_ptr() if self._events.numel() else None
        a.rope_cs, a.rope_pos0, a.rope_n = table.data_ptr(), 0, table.shape[0]
        a.cb_k, a.cb_v = cb_k.device_handle(self.device), cb_v.device_handle(self.device)
        a.strategy = int(self.config.strategy)
        _lib.check(_lib.lib.nsnkv_append(ctypes.byref(a), _stream()))
        self._keep = [k, v]  # fresh rows stay alive until the next append is enqueued
        self._cur = 1 - self._cur
        self.unit_n_chunks += n_flush
        self.unit_n_res = self.unit_n_res + n_new - n_flush * R
        self.unit_total += n_new
        return self

    def _upload(self, arr: np.ndarray) -> torch.Tensor:
        """Host array -> device tensor without a host sync: staged through a
        reused pinned buffer (a fresh pinned allocation costs ~1 ms), whose
        previous copy is fenced with an event before it is overwritten."""
        a = np.ascontiguousarray(arr)
        return _Staging.get(self.device).upload(a)

    def _as_rows(self, x) -> torch.Tensor:
        if isinstance(x, np.ndarray):
            x = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
        if not torch.is_tensor(x):
            raise ShapeMismatch("expected a tensor")
        if x.dim() == 2:
            x = x.reshape(1, 1, *x.shape)
        if x.dim() == 4:
            if x.shape[0] != self.batch or x.shape[1] != self.n_kv_heads:
                raise ShapeMismatch(f"expected [{self.batch}, {self.n_kv_heads}, n, {D}], got {tuple(x.shape)}")
            x = x.reshape(self.units, x.shape[2], x.shape[3])
        if x.dim() != 3 or x.shape[0] != self.units or x.shape[2] != D:
            raise ShapeMismatch(f"expected rows of {D} channels for {self.units} units, got {tuple(x.shape)}")
        return self._device_rows(x)

    def _as_packed(self, x, rows: int) -> torch.Tensor:
        if isinstance(x, np.ndarray):
            x = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
        if (not torch.is_tensor(x) or x.dim() != 3 or x.shape[0] != rows
                or x.shape[1] != self.n_kv_heads or x.shape[2] != D):
            raise ShapeMismatch(f"expected packed [{rows}, {self.n_kv_heads}, {D}] rows")
        return self._device_rows(x)

    def _device_rows(self, x: torch.Tensor) -> torch.Tensor:
        if x.dtype not in (torch.float32, torch.bfloat16):
            x = x.float()
        x = x.to(self.device, non_blocking=True).contiguous()
        if self.check_finite and x.numel() and not bool(torch.isfinite(x).all()):
            raise ValueError("tensor contains NaN or Inf")
        return x

    # -- sequence lifecycle ------------------------------------------------------
    def _units_of(self, seqs) -> np.ndarray:
        b = np.asarray(seqs, np.int64).reshape(-1)
        if ((b < 0) | (b >= self.batch)).any():
            raise IndexOutOfRange("sequence index out of range")
        return (b[:, None] * self.n_kv_heads + np.arange(self.n_kv_heads)[None, :]).reshape(-1)

    def release(self, seqs, base_position: int = 0) -> "PagedKvCache":
        """End sequences: their pages go back to the free list and their units
        start empty at ``base_position`` (the slot can take a new sequence)."""
        units = self._units_of(seqs)
        for u in units:
            n = int(self.unit_n_chunks[u])
            if n:
                self._free = np.concatenate([self._free, self._pt[u, :n][::-1]])
        self.unit_n_chunks[units] = 0
        self.unit_n_res[units] = 0
        self.unit_total[units] = 0
        self.unit_base[units] = int(base_position)
        ut = torch.from_numpy(units).to(self.device)
        self._cnt[self._cur][:, ut] = 0
        self.base_pos_t[ut] = int(base_position)
        return self

    def import_unit(self, unit: int, k_wire, v_wire, k_res=None, v_res=None,
                    base_position: int | None = None) -> "PagedKvCache":
        """Load one reference ``KvCacheState`` into an empty unit: serialized
        chunks (vq.py:363-380, deserialize_chunk vq.py:383-428) become pages,
        the residual rows (keys pre-RoPE, values post-HT) are copied in."""
        u = int(unit)
        if not 0 <= u < self.units:
            raise IndexOutOfRange("unit out of range")
        if self.unit_total[u]:
            raise ShapeMismatch("import_unit needs an empty unit (release it first)")
        kw, vw = list(k_wire), list(v_wire)
        if len(kw) != len(vw):
            raise ShapeMismatch("key and value chunk counts differ")
        n = len(kw)
        kr = np.zeros((0, D), np.float32) if k_res is None else np.array(k_res, np.float32).reshape(-1, D)
        vr = np.zeros((0, D), np.float32) if v_res is None else np.array(v_res, np.float32).reshape(-1, D)
        if kr.shape != vr.shape or kr.shape[0] >= R:
            raise ShapeMismatch("residual rows must be [< 64, 128] for keys and values alike")
        for blob in kw + vw:
            _n, _d, bm, strat = struct.unpack_from("<HHBB", bytes(blob), 0)
            if bm != int(self.bit_mode) or strat != int(self.config.strategy):
                raise FormatError("chunk bit mode / strategy does not match the cache")
        if base_position is not None:
            self.unit_base[u] = int(base_position)
            self.base_pos_t[u] = int(base_position)
        if n:
            ids = self._alloc(n)
            self._ensure_width(n)
            self._pt[u, :n] = ids
            for kind, blobs in (("k", kw), ("v", vw)):
                pages = np.stack([wire_to_page(bytes(b), kind) for b in blobs])
                _lib.check(_lib.lib.nsnkv_pages_copy(self._pools[kind].ptr, self.page_bytes,
                                                     ids.ctypes.data, n, pages.ctypes.data, 1, _stream()))
            self.page_table[u, :n] = torch.from_numpy(ids).to(self.device)
            self._events[torch.from_numpy(ids.astype(np.int64)).to(self.device)] = 0
            torch.cuda.current_stream(self.device).synchronize()  # host page buffers
        m = kr.shape[0]
        if m:
            self.k_res[u, :m] = torch.from_numpy(kr).to(self.device)
            self.v_res[u, :m] = torch.from_numpy(vr).to(self.device)
        self._cnt[self._cur, 0, u] = n
        self._cnt[self._cur, 1, u] = m
        self.unit_n_chunks[u], self.unit_n_res[u], self.unit_total[u] = n, m, n * R + m
        self.rope.ensure(int(self.unit_base[u]) + n * R + R)
        return self

    def load_snapshot(self, unit: int, blob: bytes) -> "PagedKvCache":
        """Inverse of ``snapshot`` / the reference kvcache.snapshot byte image
        (kvcache.py:198-213)."""
        b = bytes(blob)
        if b[:4] != b"NSNS":
            raise FormatError("bad snapshot: missing magic")
        n, total, base = struct.unpack_from("<IQQ", b, 4)
        pos = 24
        blobs = []
        for _ in range(2 * n):
            (ln,) = struct.unpack_from("<I", b, pos)
            blobs.append(b[pos + 4:pos + 4 + ln])
            pos += 4 + ln
        res = []
        for _ in range(2):
            (ln,) = struct.unpack_from("<I", b, pos)
            t = b[pos + 4:pos + 4 + ln]
            pos += 4 + ln
            if t[:4] != b"NSNT":
                raise FormatError("bad snapshot: residual tensor")
            rows, cols = struct.unpack_from("<II", t, 4)
            res.append(np.frombuffer(t, "<f4", rows * cols, 12).reshape(rows, cols))
        if pos != len(b):
            raise FormatError("bad snapshot: trailing bytes")
        if total != n * R + res[0].shape[0]:
            raise FormatError("bad snapshot: token count")
        return self.import_unit(unit, blobs[:n], blobs[n:], res[0], res[1], base_position=base)

    # -- decode ----------------------------------------------------------------
    def view(self, n_q_heads: int, cb_k: Codebook | None = None,
             cb_v: Codebook | None = None) -> _lib.CacheView:
        cb_k = cb_k or self.cb_k
        cb_v = cb_v or self.cb_v
        if cb_k is None or cb_v is None:
            raise ShapeMismatch("decode needs the key and value codebooks")
        if n_q_heads % self.n_kv_heads:
            raise ShapeMismatch("n_q_heads must be a multiple of n_kv_heads")
        table = self.rope.ensure(int((self.unit_base + self.unit_n_chunks * R).max()) + R)
        cnt = self._cnt[self._cur]
        cv = _lib.CacheView()
        cv.k_pool, cv.v_pool = self.pool_ptrs()
        cv.page_table = self.page_table.data_ptr() if self.page_table.numel() else None
        cv.page_table_stride = self.page_table.stride(0) if self.page_table.numel() else 0
        cv.n_chunks = cnt[0].data_ptr()
        cv.k_res = self.k_res.data_ptr()
        cv.v_res = self.v_res.data_ptr()
        cv.n_res = cnt[1].data_ptr()
        cv.base_pos = self.base_pos_t.data_ptr()
        cv.batch = self.batch
        cv.n_kv_heads = self.n_kv_heads
        cv.n_q_heads = n_q_heads
        cv.max_tokens = self.max_tokens
        cv.rope_cs = table.data_ptr()
        cv.rope_pos0 = 0
        cv.rope_n = table.shape[0]
        cv.cb_k = cb_k.device_handle(self.device)
        cv.cb_v = cb_v.device_handle(self.device)
        cv.total_chunks = int(self.unit_n_chunks.sum())
        cv.precision = PRECISIONS[self.precision]
        return cv

    def _q(self, q) -> torch.Tensor:
        if isinstance(q, np.ndarray):
            q = torch.from_numpy(np.ascontiguousarray(q, dtype=np.float32))
        q = q.to(self.device, torch.float32).contiguous()
        if q.dim() == 1:
            q = q.reshape(1, 1, D)
        if q.dim() != 3 or q.shape[0] != self.batch or q.shape[2] != D:
            raise ShapeMismatch(f"query must be [{self.batch}, n_q_heads, {D}], got {tuple(q.shape)}")
        return q

    def _workspace(self, cv) -> torch.Tensor:
        need = int(_lib.lib.nsnkv_decode_workspace_bytes(cv))
        if self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device=self.device)
        return self._ws

    def scores(self, q, cb_k: Codebook | None = None) -> torch.Tensor:
        """Raw q.K^T [B, Hq, total_tokens] (attention.py:83-111)."""
        q = self._q(q)
        cv = self.view(q.shape[1], cb_k=cb_k)
        out = torch.empty(self.batch, q.shape[1], cv.max_tokens, dtype=torch.float32, device=self.device)
        if self.total_tokens:
            _lib.check(_lib.lib.nsnkv_decode_scores(cv, q.data_ptr(), out.data_ptr(), _stream()))
        return out[:, :, :self.total_tokens]

    def output(self, weights, n_q_heads: int | None = None,
               cb_v: Codebook | None = None) -> torch.Tensor:
        """Weighted value sum in the model basis [B, Hq, 128] (attention.py:114-133)."""
        if isinstance(weights, np.ndarray):
            weights = torch.from_numpy(np.ascontiguousarray(weights, dtype=np.float32))
        w = weights.to(self.device, torch.float32)
        if w.dim() == 1:
            w = w.reshape(1, 1, -1)
        if w.shape[-1] != self.total_tokens:
            raise ShapeMismatch(f"{w.shape[-1]} weights for {self.total_tokens} cached tokens")
        hq = w.shape[1] if n_q_heads is None else n_q_heads
        cv = self.view(hq, cb_v=cb_v)
        wp = torch.zeros(self.batch, hq, cv.max_tokens, dtype=torch.float32, device=self.device)
        wp[:, :, :self.total_tokens] = w
        out = torch.empty(self.batch, hq, D, dtype=torch.float32, device=self.device)
        ws = self._workspace(cv)
        _lib.check(_lib.lib.nsnkv_decode_output(cv, wp.data_ptr(), out.data_ptr(), ws.data_ptr(),
                                                ws.numel(), _stream()))
        return out

    def attend(self, q, out: torch.Tensor | None = None, lse: torch.Tensor | None = None) -> torch.Tensor:
        """Fused softmax(q.K^T / sqrt(d)) . V -> [B, Hq, 128] (attention.py:136-142)."""
        if self.total_tokens == 0:
            raise ShapeMismatch("attention over an empty cache")
        q, cv, out = self._attend_args(q, out, lse)
        ws = self._workspace(cv)
        _lib.check(_lib.lib.nsnkv_decode_attend(cv, q.data_ptr(), out.data_ptr(),
                                                lse.data_ptr() if lse is not None else None,
                                                ws.data_ptr(), ws.numel(), _stream()))
        return out

    def _attend_args(self, q, out, lse):
        q = self._q(q)
        cv = self.view(q.shape[1])
        rows = self.batch * q.shape[1]
        if out is None:
            out = torch.empty(self.batch, q.shape[1], D, dtype=torch.float32, device=self.device)
        # the kernels write fp32 [B*Hq, 128] / [B*Hq] through raw pointers
        for name, t, n in (("out", out, rows * D), ("lse", lse, rows)):
            if t is None:
                continue
            if (t.dtype != torch.float32 or not t.is_contiguous() or t.device != self.device
                    or t.numel() != n):
                raise ShapeMismatch(f"{name} must be a contiguous float32 tensor of {n} elements "
                                    f"on {self.device}, got {t.dtype} {tuple(t.shape)} on {t.device}")
        return q, cv, out

    def decode_step(self, q, keys, values, out: torch.Tensor | None = None,
                    lse: torch.Tensor | None = None) -> torch.Tensor:
        """One serving decode step: append [B, H_kv, n, 128] keys / values
        (n >= 1, usually 1) to every sequence, then attend q over the cache
        including them (kvcache.append + attend_quantized).  When no unit
        completes a chunk this is the attend launches alone (the combine
        kernel attends the new rows as residual rows and stores them); a step
        that completes a chunk runs nsnkv_append first."""
        k = self._as_rows(keys)
        v = self._as_rows(values)
        if k.shape != v.shape:
            raise ShapeMismatch("key and value batches must have the same shape")
        n = k.shape[1]
        if n < 1 or int((self.unit_n_res + n).max()) >= R:
            self.append(k, v)
            return self.attend(q, out=out, lse=lse)
        if k.dtype != v.dtype:
            k, v = k.float(), v.float()
        q, cv, out = self._attend_args(q, out, lse)
        ws = self._workspace(cv)
        _lib.check(_lib.lib.nsnkv_decode_step(
            cv, q.data_ptr(), k.data_ptr(), v.data_ptr(), 1 if k.dtype == torch.bfloat16 else 0, n,
            self._cnt[self._cur][1].data_ptr(), out.data_ptr(),
            lse.data_ptr() if lse is not None else None, ws.data_ptr(), ws.numel(), _stream()))
        self._keep = [k, v]
        self.unit_n_res += n
        self.unit_total += n
        return out

    # -- counters (kvcache.py:86-88, 191-194) ---------------------------------
    def counters(self) -> np.ndarray:
        """Per-unit [clamp, zero_vector, s3_fallback, near_tie] event totals."""
        ev = self._events.sum(dim=1).cpu().numpy().astype(np.int64)  # [page][4], K + V
        out = np.zeros((self.units, 4), np.int64)
        for u in range(self.units):
            n = int(self.unit_n_chunks[u])
            if n:
                out[u] = ev[self._pt[u, :n]].sum(axis=0)
        return out

    # -- export: pages -> reference wire format (vq.py:363-380) ---------------
    def pages(self, unit: int, kind: str = "k") -> np.ndarray:
        """[n_chunks, page_bytes] device pages of one unit (host copy)."""
        n = int(self.unit_n_chunks[unit])
        out = np.empty((n, self.page_bytes), np.uint8)
        if n:
            ids = np.ascontiguousarray(self._pt[unit, :n])
            _lib.check(_lib.lib.nsnkv_pages_copy(self._pools[kind].ptr, self.page_bytes,
                                                 ids.ctypes.data, n, out.ctypes.data, 0, _stream()))
            torch.cuda.current_stream(self.device).synchronize()
        return out

    def all_pages(self, kind: str = "k") -> np.ndarray:
        """Pages of every unit, unit-major ([sum n_chunks, page_bytes])."""
        ids = np.concatenate([self._pt[u, :self.unit_n_chunks[u]] for u in range(self.units)]
                             ).astype(np.int32)
        out = np.empty((ids.size, self.page_bytes), np.uint8)
        if ids.size:
            _lib.check(_lib.lib.nsnkv_pages_copy(self._pools[kind].ptr, self.page_bytes,
                                                 ids.ctypes.data, ids.size, out.ctypes.data, 0,
                                                 _stream()))
            torch.cuda.current_stream(self.device).synchronize()
        return out

    def wire_chunks(self, unit: int, kind: str = "k") -> np.ndarray:
        """[n_chunks, wire_bytes] reference serialized chunks of one unit."""
        return pages_to_wire(self.pages(unit, kind), self.bit_mode, self.config.strategy, kind)

    def chunk_wire(self, unit: int, kind: str = "k") -> list[bytes]:
        return [w.tobytes() for w in self.wire_chunks(unit, kind)]

    def snapshot(self, unit: int = 0) -> bytes:
        """kvcache.snapshot byte image of one unit (kvcache.py:198-213)."""
        n, m = int(self.unit_n_chunks[unit]), int(self.unit_n_res[unit])
        out = bytearray(b"NSNS")
        out += struct.pack("<IQQ", n, int(self.unit_total[unit]), int(self.unit_base[unit]))
        for kind in ("k", "v"):
            for blob in self.chunk_wire(unit, kind):
                out += struct.pack("<I", len(blob)) + blob
        for res in (self.k_res, self.v_res):
            rows = res[unit, :m].cpu().numpy().astype("<f4")
            blob = b"NSNT" + struct.pack("<II", rows.shape[0], D) + rows.tobytes()
            out += struct.pack("<I", len(blob)) + blob
        return bytes(out)


# ---------------------------------------------------------------------------
# page <-> wire conversion (host side, numpy)
# ---------------------------------------------------------------------------
_LAYOUT = {  # idx, sgn, s2, s1n, on, par
    BitMode.TWO_BIT: (0, 1024, 2048, 2176, 2208, 2272),
    BitMode.ONE_BIT: (0, -1, 1024, 1152, 1184, 1248),
}


def unpermute_signs(words: np.ndarray) -> np.ndarray:
    """[..., 64, 4] u32 decode-order sign words -> natural sign bytes [..., 64, 16].
    Word q of a token covers subs 4q+m; bit 4m+p holds the sign of component
    2p and bit 16+4m+p the sign of component 2p+1 (see csrc/common.cuh)."""
    w = words.astype(np.uint32)
    out = np.zeros(w.shape[:-1] + (16,), np.uint32)
    for q in range(4):
        for m in range(4):
            for p in range(4):
                out[..., 4 * q + m] |= ((w[..., q] >> (4 * m + p)) & 1) << (2 * p)
                out[..., 4 * q + m] |= ((w[..., q] >> (16 + 4 * m + p)) & 1) << (2 * p + 1)
    return out.astype(np.uint8)


def permute_signs(signs: np.ndarray) -> np.ndarray:
    """Natural sign bytes [..., 64, 16] -> decode-order words [..., 64, 4] u32."""
    s = signs.astype(np.uint32)
    words = np.zeros(s.shape[:-1] + (4,), np.uint32)
    for q in range(4):
        for m in range(4):
            for p in range(4):
                words[..., q] |= ((s[..., 4 * q + m] >> (2 * p)) & 1) << (4 * m + p)
                words[..., q] |= ((s[..., 4 * q + m] >> (2 * p + 1)) & 1) << (16 + 4 * m + p)
    return words


def unpermute_signs_v(words: np.ndarray) -> np.ndarray:
    """[..., 256] u32 value-page sign words -> natural sign bytes [..., 64, 16].
    Word 8 i + c holds component c of token pair (2i, 2i+1): bit j = token
    2i, sub j; bit 16 + j = token 2i+1 (see csrc/encode.cu)."""
    w = words.astype(np.uint32).reshape(words.shape[:-1] + (32, 8))
    out = np.zeros(words.shape[:-1] + (32, 2, 16), np.uint32)
    for c in range(8):
        for j in range(16):
            out[..., 0, j] |= ((w[..., c] >> j) & 1) << c
            out[..., 1, j] |= ((w[..., c] >> (16 + j)) & 1) << c
    return out.reshape(words.shape[:-1] + (64, 16)).astype(np.uint8)


def permute_signs_v(signs: np.ndarray) -> np.ndarray:
    """Natural sign bytes [..., 64, 16] -> value-page words [..., 256] u32."""
    s = signs.astype(np.uint32).reshape(signs.shape[:-2] + (32, 2, 16))
    w = np.zeros(signs.shape[:-2] + (32, 8), np.uint32)
    for c in range(8):
        for j in range(16):
            w[..., c] |= ((s[..., 0, j] >> c) & 1) << j
            w[..., c] |= ((s[..., 1, j] >> c) & 1) << (16 + j)
    return w.reshape(signs.shape[:-2] + (256,))


def wire_bytes(bit_mode) -> int:
    """Bytes of one serialized chunk (vq.py:363-380)."""
    return 6 + 1024 + (1024 if int(bit_mode) == 2 else 0) + 36 + 80 + 128


def pages_to_wire(pages: np.ndarray, bit_mode, strategy, kind: str = "k") -> np.ndarray:
    """[n, page_bytes] device pages -> [n, wire_bytes] reference serialized
    chunks (vq.py:363-380), vectorised over chunks.  kind "k" / "v": key and
    value pages order their sign bits for their own decode side."""
    bm = BitMode(bit_mode)
    o_idx, o_sgn, o_s2, o_s1n, o_on, o_par = _LAYOUT[bm]
    p = np.ascontiguousarray(pages, dtype=np.uint8).reshape(-1, PAGE_BYTES[bm])
    n = p.shape[0]
    out = np.empty((n, wire_bytes(bm)), np.uint8)
    out[:, :6] = np.frombuffer(struct.pack("<HHBB", R, D, int(bm), int(strategy)), np.uint8)
    pos = 6
    out[:, pos:pos + 1024] = p[:, o_idx:o_idx + 1024]
    pos += 1024
    if bm is BitMode.TWO_BIT:
        w = p[:, o_sgn:o_sgn + 1024].copy().view("<u4")
        nat = unpermute_signs(w.reshape(n, R, 4)) if kind == "k" else unpermute_signs_v(w)
        out[:, pos:pos + 1024] = nat.reshape(n, 1024)
        pos += 1024
    par = p[:, o_par:o_par + 20]
    out[:, pos:pos + 4] = par[:, 0:4]                       # s1 scale, zero
    pos += 4
    out[:, pos:pos + 32] = p[:, o_s1n:o_s1n + 32]
    pos += 32
    for g in range(4):                                      # (o scale, o zero) per group
        out[:, pos:pos + 2] = par[:, 4 + 2 * g:6 + 2 * g]
        out[:, pos + 2:pos + 4] = par[:, 12 + 2 * g:14 + 2 * g]
        pos += 4
    out[:, pos:pos + 64] = p[:, o_on:o_on + 64]
    pos += 64
    out[:, pos:pos + 128] = p[:, o_s2:o_s2 + 128]
    return out


def page_to_wire(page: np.ndarray, bit_mode: BitMode, strategy: ScaleStrategy,
                 kind: str = "k") -> bytes:
    return pages_to_wire(np.asarray(page)[None], bit_mode, strategy, kind)[0].tobytes()


def wire_to_page(blob: bytes, kind: str = "k") -> np.ndarray:
    """Inverse of page_to_wire (for loading reference-serialized chunks)."""
    n, d, bm_raw, _strategy = struct.unpack_from("<HHBB", blob, 0)
    if n != R or d != D:
        raise Unsupported("GPU pages hold 64 x 128 chunks")
    bm = BitMode(bm_raw)
    o_idx, o_sgn, o_s2, o_s1n, o_on, o_par = _LAYOUT[bm]
    page = np.zeros(PAGE_BYTES[bm], np.uint8)
    b = np.frombuffer(blob, np.uint8)
    pos = 6
    page[o_idx:o_idx + 1024] = b[pos:pos + 1024]
    pos += 1024
    if bm is BitMode.TWO_BIT:
        nat = b[pos:pos + 1024].reshape(R, 16)
        words = permute_signs(nat) if kind == "k" else permute_signs_v(nat)
        page[o_sgn:o_sgn + 1024] = words.astype("<u4").view(np.uint8).ravel()
        pos += 1024
    par = np.zeros(10, "<u2")
    par[0], par[1] = struct.unpack_from("<HH", blob, pos)
    pos += 4
    page[o_s1n:o_s1n + 32] = b[pos:pos + 32]
    pos += 32
    for g in range(4):
        par[2 + g], par[6 + g] = struct.unpack_from("<HH", blob, pos)
        pos += 4
    page[o_on:o_on + 64] = b[pos:pos + 64]
    pos += 64
    page[o_s2:o_s2 + 128] = b[pos:pos + 128]
    page[o_par:o_par + 20] = par.view(np.uint8)
    return page


def ledger_bytes(bit_mode) -> int:
    """Bytes per chunk from the reference bit ledger (vq.py:328-356)."""
    return LEDGER_BYTES[BitMode.parse(bit_mode)]


def avg_bits_per_value(bit_mode) -> float:
    return ledger_bytes(bit_mode) * 8 / (R * D)


def inv_sqrt_d() -> float:
    return 1.0 / math.sqrt(D)
