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
``KvCacheState`` each) in device memory: packed pages for every flushed
64-token chunk (K and V pools), a page table, and the fp32 residual rows.
Every unit of a batch advances by the same token count per ``append`` (the
serving case: one decode token or one prefill block per sequence); the
single-head facade in ``api.py`` is a 1 x 1 batch.
"""

from __future__ import annotations

import os

import enum
import math
import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .codebook import BitMode, Codebook
from .errors import ShapeMismatch, Unsupported

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
    4K context: 3e-2).  Value codewords may be plain fp16 in
    2-bit mode ("vfast": the per-component signs make the rounding errors
    cancel, <= 2.5e-4 at 32K context), but not in 1-bit mode, where the
    unsigned codewords accumulate a bias that grows with the context (1.5e-3
    at 4K, 3.7e-3 at 32K), so 1-bit decodes "precise"."""
    return "vfast" if int(bit_mode) == 2 else "precise"


def check_precision(precision: str, bit_mode, allow_inexact: bool = False) -> str:
    """Validate a precision mode for a bit mode.  Modes that are known to
    exceed the 1e-3 output tolerance on some inputs ("fast" in either bit
    mode, "vfast" in 1-bit mode) need an explicit allow_inexact=True."""
    if precision not in PRECISIONS:
        raise ValueError(f"precision must be one of {sorted(PRECISIONS)}")
    inexact = precision == "fast" or (precision == "vfast" and int(bit_mode) == 1)
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
class PagedKvCache:
    """B x H_kv units of packed KV cache on one GPU (see module docstring)."""

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
        self.total_tokens = 0
        self.n_chunks = 0
        self.n_res = 0
        self.max_chunks = 0
        dev = self.device
        self.k_res = torch.zeros(self.units, R, D, dtype=torch.float32, device=dev)
        self.v_res = torch.zeros(self.units, R, D, dtype=torch.float32, device=dev)
        self.base_pos_t = torch.full((self.units,), self.base_position, dtype=torch.int64, device=dev)
        self.k_pool = torch.zeros(0, self.page_bytes, dtype=torch.uint8, device=dev)
        self.v_pool = torch.zeros(0, self.page_bytes, dtype=torch.uint8, device=dev)
        self.page_table = torch.zeros(self.units, 0, dtype=torch.int32, device=dev)
        self.k_counters = torch.zeros(self.units, 0, 4, dtype=torch.int32, device=dev)
        self.v_counters = torch.zeros(self.units, 0, 4, dtype=torch.int32, device=dev)
        self._n_chunks_t = torch.zeros(self.units, dtype=torch.int32, device=dev)
        self._n_res_t = torch.zeros(self.units, dtype=torch.int32, device=dev)
        self._ws = torch.empty(0, dtype=torch.uint8, device=dev)
        self.rope = RopeTable.get(dev, config.rope_base)
        self._reserve_chunks((max_tokens + R - 1) // R)

    # -- storage ------------------------------------------------------------
    def _reserve_chunks(self, n: int) -> None:
        """Grow the page pools so every unit can hold n chunks (pages of unit
        u are u * max_chunks .. u * max_chunks + max_chunks - 1)."""
        if n <= self.max_chunks:
            return
        new = max(n, 2 * self.max_chunks)
        dev = self.device
        kp = torch.zeros(self.units * new, self.page_bytes, dtype=torch.uint8, device=dev)
        vp = torch.zeros_like(kp)
        kc = torch.zeros(self.units, new, 4, dtype=torch.int32, device=dev)
        vc = torch.zeros_like(kc)
        if self.max_chunks:
            old = self.max_chunks
            kp.view(self.units, new, -1)[:, :old].copy_(self.k_pool.view(self.units, old, -1))
            vp.view(self.units, new, -1)[:, :old].copy_(self.v_pool.view(self.units, old, -1))
            kc[:, :old].copy_(self.k_counters)
            vc[:, :old].copy_(self.v_counters)
        self.k_pool, self.v_pool, self.k_counters, self.v_counters = kp, vp, kc, vc
        self.page_table = (torch.arange(self.units, device=dev, dtype=torch.int32)[:, None] * new
                           + torch.arange(new, device=dev, dtype=torch.int32)[None, :]).contiguous()
        self.max_chunks = new

    def reserve(self, max_tokens: int) -> "PagedKvCache":
        """Pre-size the page pools and the RoPE table for contexts up to
        max_tokens per unit, so later appends never grow them (a growth
        reallocates and copies the pools: a server reserves up front)."""
        n = (int(max_tokens) + R - 1) // R
        if n > self.max_chunks:
            self._reserve_chunks(n)
        self.rope.ensure(self.base_position + n * R)
        return self

    @property
    def n_quantized(self) -> int:
        return self.n_chunks * R

    @property
    def max_tokens(self) -> int:
        """Row stride of score / weight buffers (a multiple of 64)."""
        return max(R, (self.n_chunks + (1 if self.n_res else 0)) * R)

    # -- append (kvcache.py:157-195) ------------------------------------------
    def append(self, keys, values, cb_k: Codebook | None = None,
               cb_v: Codebook | None = None) -> "PagedKvCache":
        """Append [B, H_kv, n, 128] keys (pre-RoPE) and values (post-HT)."""
        cb_k = cb_k or self.cb_k
        cb_v = cb_v or self.cb_v
        if cb_k is None or cb_v is None:
            raise ShapeMismatch("append needs the key and value codebooks")
        if cb_k.bit_mode != self.bit_mode or cb_v.bit_mode != self.bit_mode:
            raise ShapeMismatch("codebook bit mode does not match the cache")
        self.cb_k, self.cb_v = cb_k, cb_v
        k = self._as_rows(keys)
        v = self._as_rows(values)
        if k.shape != v.shape:
            raise ShapeMismatch("key and value batches must have the same shape")
        if k.dtype != v.dtype:  # one fp32 / one bf16 batch: encode both from fp32
            k, v = k.float(), v.float()
        n = k.shape[1]
        if n < 1:
            raise ShapeMismatch("append needs at least one token")
        n_flush = (self.n_res + n) // R
        if n_flush:
            self._reserve_chunks(self.n_chunks + n_flush)
            start = self.base_position + self.n_chunks * R
            table = self.rope.ensure(start + n_flush * R)
            page_ids = self.page_table[:, self.n_chunks:]
            start_t = self._start_pos(start)
            for is_key, rows, res, pool, cb, cnt in (
                    (1, k, self.k_res, self.k_pool, cb_k, self.k_counters),
                    (0, v, self.v_res, self.v_pool, cb_v, self.v_counters)):
                cnt_view = cnt[:, self.n_chunks:self.n_chunks + n_flush]
                cnt_buf = torch.empty(self.units, n_flush, 4, dtype=torch.int32, device=self.device)
                _lib.check(_lib.lib.nsnkv_encode_chunks(
                    res.data_ptr(), self.n_res, rows.data_ptr(),
                    1 if rows.dtype == torch.bfloat16 else 0, n, self.units, n_flush,
                    is_key, start_t.data_ptr(),
                    table.data_ptr(), 0, table.shape[0], cb.device_handle(self.device),
                    int(self.config.strategy), pool.data_ptr(), page_ids.data_ptr(),
                    self.page_table.stride(0), cnt_buf.data_ptr(), _stream()))
                cnt_view.copy_(cnt_buf)
        # the residual keeps stream rows [n_flush * R, n_res + n)
        consumed_fresh = n_flush * R - self.n_res if n_flush else 0
        keep_from_res = 0 if n_flush else self.n_res
        tail = n - consumed_fresh
        if tail:
            for rows, res in ((k, self.k_res), (v, self.v_res)):
                res[:, keep_from_res:keep_from_res + tail].copy_(rows[:, consumed_fresh:])
        self.n_res = keep_from_res + tail
        self.n_chunks += n_flush
        self.total_tokens += n
        self._n_chunks_t.fill_(self.n_chunks)
        self._n_res_t.fill_(self.n_res)
        return self

    def _start_pos(self, start: int) -> torch.Tensor:
        return torch.full((self.units,), start, dtype=torch.int64, device=self.device)

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
        if x.dtype not in (torch.float32, torch.bfloat16):
            x = x.float()
        x = x.to(self.device, non_blocking=True).contiguous()
        if self.check_finite and x.numel() and not bool(torch.isfinite(x).all()):
            raise ValueError("tensor contains NaN or Inf")
        return x

    # -- decode ----------------------------------------------------------------
    def view(self, n_q_heads: int, cb_k: Codebook | None = None,
             cb_v: Codebook | None = None) -> _lib.CacheView:
        cb_k = cb_k or self.cb_k
        cb_v = cb_v or self.cb_v
        if cb_k is None or cb_v is None:
            raise ShapeMismatch("decode needs the key and value codebooks")
        if n_q_heads % self.n_kv_heads:
            raise ShapeMismatch("n_q_heads must be a multiple of n_kv_heads")
        table = self.rope.ensure(self.base_position + self.n_chunks * R + R)
        cv = _lib.CacheView()
        cv.k_pool = self.k_pool.data_ptr()
        cv.v_pool = self.v_pool.data_ptr()
        cv.page_table = self.page_table.data_ptr()
        cv.page_table_stride = self.page_table.stride(0)
        cv.n_chunks = self._n_chunks_t.data_ptr()
        cv.k_res = self.k_res.data_ptr()
        cv.v_res = self.v_res.data_ptr()
        cv.n_res = self._n_res_t.data_ptr()
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
        cv.total_chunks = self.units * self.n_chunks
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
        q = self._q(q)
        if self.total_tokens == 0:
            raise ShapeMismatch("attention over an empty cache")
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
        ws = self._workspace(cv)
        _lib.check(_lib.lib.nsnkv_decode_attend(cv, q.data_ptr(), out.data_ptr(),
                                                lse.data_ptr() if lse is not None else None,
                                                ws.data_ptr(), ws.numel(), _stream()))
        return out

    # -- counters (kvcache.py:86-88, 191-194) ---------------------------------
    def counters(self) -> np.ndarray:
        """Per-unit [clamp, zero_vector, s3_fallback, near_tie] event totals."""
        k = self.k_counters[:, :self.n_chunks].sum(dim=1)
        v = self.v_counters[:, :self.n_chunks].sum(dim=1)
        return (k + v).cpu().numpy().astype(np.int64)

    # -- export: pages -> reference wire format (vq.py:363-380) ---------------
    def pages(self, unit: int, kind: str = "k") -> np.ndarray:
        pool = self.k_pool if kind == "k" else self.v_pool
        ids = self.page_table[unit, :self.n_chunks].long()
        return pool[ids].cpu().numpy()

    def wire_chunks(self, unit: int, kind: str = "k") -> np.ndarray:
        """[n_chunks, wire_bytes] reference serialized chunks of one unit."""
        return pages_to_wire(self.pages(unit, kind), self.bit_mode, self.config.strategy, kind)

    def chunk_wire(self, unit: int, kind: str = "k") -> list[bytes]:
        return [w.tobytes() for w in self.wire_chunks(unit, kind)]

    def snapshot(self, unit: int = 0) -> bytes:
        """kvcache.snapshot byte image of one unit (kvcache.py:198-213)."""
        out = bytearray(b"NSNS")
        out += struct.pack("<IQQ", self.n_chunks, self.total_tokens, self.base_position)
        for kind in ("k", "v"):
            for blob in self.chunk_wire(unit, kind):
                out += struct.pack("<I", len(blob)) + blob
        for res in (self.k_res, self.v_res):
            rows = res[unit, :self.n_res].cpu().numpy().astype("<f4")
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
