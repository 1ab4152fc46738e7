"""Reference pipeline API (single KV head), backed by the GPU cache.

Drop-in for the reference's level-2 functions (re-exported by
pkg/src/nsnkv/__init__.py:12-63):
  new_cache(config, base_position)                  kvcache.py:110
  append(state, keys, values, cb_k, cb_v)           kvcache.py:157-195
  scores_quantized(q_roped, state, cb_k)            attention.py:83-111
  output_quantized(weights, state, cb_v)            attention.py:114-133
  attend_quantized(q_roped, state, cb_k, cb_v)      attention.py:136-142
  snapshot(state)                                   kvcache.py:198-213
Inputs and outputs are host numpy arrays like the reference's; the work runs
in the CUDA kernels of libnsnkv_b200.so.  ``KvCacheState`` is a 1 x 1
``PagedKvCache`` and exposes the reference state fields the callers read.
"""

from __future__ import annotations

import numpy as np
import torch

from .cache import CacheConfig, PagedKvCache
from .codebook import Codebook
from .errors import ShapeMismatch


class KvCacheState:
    """One (sequence, kv-head) cache (reference kvcache.py:77-107)."""

    def __init__(self, config: CacheConfig, base_position: int = 0):
        self.config = config
        self.gpu = PagedKvCache(config, 1, 1, cb_k=None, cb_v=None, base_position=base_position)

    # reference fields -------------------------------------------------------
    @property
    def total_tokens(self) -> int:
        return self.gpu.total_tokens

    @property
    def base_position(self) -> int:
        return self.gpu.base_position

    @property
    def n_quantized(self) -> int:
        return self.gpu.n_quantized

    @property
    def n_chunks(self) -> int:
        return self.gpu.n_chunks

    @property
    def residual_count(self) -> int:
        return self.gpu.n_res

    @property
    def residual_positions(self) -> np.ndarray:
        return self.base_position + np.arange(self.n_quantized, self.total_tokens)

    def _counter(self, i: int) -> int:
        return int(self.gpu.counters()[0, i])

    @property
    def clamp_count(self) -> int:
        return self._counter(0)

    @property
    def zero_vector_count(self) -> int:
        return self._counter(1)

    @property
    def s3_fallback_count(self) -> int:
        return self._counter(2)

    @property
    def near_tie_count(self) -> int:
        """Sub-vectors whose argmax needed the exact fp64 re-score."""
        return self._counter(3)

    def key_residual_tokens(self) -> np.ndarray:
        return self.gpu.k_res[0, :self.gpu.n_res].cpu().numpy()

    def value_residual_tokens(self) -> np.ndarray:
        return self.gpu.v_res[0, :self.gpu.n_res].cpu().numpy()

    def key_chunk_wire(self) -> list[bytes]:
        return self.gpu.chunk_wire(0, "k")

    def value_chunk_wire(self) -> list[bytes]:
        return self.gpu.chunk_wire(0, "v")


def new_cache(config: CacheConfig, base_position: int = 0) -> KvCacheState:
    return KvCacheState(config, base_position)


def _rows(x, d: int) -> np.ndarray:
    a = np.ascontiguousarray(x, dtype=np.float32)
    if a.ndim != 2:
        raise ShapeMismatch(f"expected 2-D tensor, got ndim={a.ndim}")
    if a.shape[1] != d:
        raise ShapeMismatch(f"expected {d} channels, got {a.shape[1]}")
    if a.size and not np.isfinite(a).all():
        raise ValueError("tensor contains NaN or Inf")
    return a


def append(state: KvCacheState, new_keys, new_values, cb_k: Codebook, cb_v: Codebook) -> KvCacheState:
    """Keys pre-RoPE, values post-Hadamard (kvcache.py:157-195)."""
    d = state.config.d
    k = _rows(new_keys, d)
    v = _rows(new_values, d)
    if k.shape != v.shape:
        raise ShapeMismatch("key and value batches must have the same shape")
    if k.shape[0] < 1:
        raise ShapeMismatch("append needs at least one token")
    state.gpu.append(k[None, None], v[None, None], cb_k, cb_v)
    return state


def _query(q_roped, d: int) -> np.ndarray:
    q = np.ascontiguousarray(q_roped, dtype=np.float32).reshape(-1)
    if q.shape[0] != d:
        raise ShapeMismatch(f"query has dim {q.shape[0]}, cache has {d}")
    return q


def scores_quantized(q_roped, state: KvCacheState, cb_k: Codebook) -> np.ndarray:
    q = _query(q_roped, state.config.d)
    if state.total_tokens == 0:
        return np.zeros(0, dtype=np.float32)
    s = state.gpu.scores(q.reshape(1, 1, -1), cb_k=cb_k)
    return s[0, 0].cpu().numpy()


def output_quantized(weights, state: KvCacheState, cb_v: Codebook) -> np.ndarray:
    w = np.asarray(weights, dtype=np.float32).reshape(-1)
    if w.shape[0] != state.total_tokens:
        raise ShapeMismatch(f"{w.shape[0]} weights for {state.total_tokens} cached tokens")
    out = state.gpu.output(w.reshape(1, 1, -1), n_q_heads=1, cb_v=cb_v)
    return out[0, 0].cpu().numpy()


def attend_quantized(q_roped, state: KvCacheState, cb_k: Codebook, cb_v: Codebook):
    """(weights, output) like the reference: scores on the GPU, fp64 softmax of
    scores / sqrt(d) (attention.py:46-50, 141), then the GPU weighted sum."""
    q = _query(q_roped, state.config.d)
    s = state.gpu.scores(q.reshape(1, 1, -1), cb_k=cb_k)[0, 0]
    z = s.double() / float(np.sqrt(state.config.d))
    w = torch.softmax(z, dim=-1).float()
    out = state.gpu.output(w.reshape(1, 1, -1), n_q_heads=1, cb_v=cb_v)
    return w.cpu().numpy(), out[0, 0].cpu().numpy()


def snapshot(state: KvCacheState) -> bytes:
    return state.gpu.snapshot(0)
