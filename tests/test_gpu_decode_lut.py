"""1-bit decode with the key side by lookup table (attend3_kernel PREC 3:
LUT[c][j] = <HT(q_h)_j, e_c> for the unit's 4 q-heads, built in shared memory
at every unit change of a CTA's chunk range; reference attention.py:96-104).
The dispatcher takes this path for 1-bit, G = 4, "vfast" when the CTAs' ranges
hold >= 32 chunks on average; NSNKV_NO_LUT=1 selects the gather path instead.

Checked against the oracle (reference attention.py:136-142 restated) on
ragged batches where every CTA crosses several units, empty units included,
and on misaligned (outlier) data at BASELINE length.  Tolerance: max|d out| <=
1e-3 * max|out| per (batch, q-head), the north-star bound."""

from __future__ import annotations

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-3


def _oracle(cache, unit, n, q_unit):
    from oracle import oracle as orc

    oc = orc.OracleCache(cache.cb_k.entries, cache.cb_v.entries, int(cache.cb_k.bit_mode),
                         base_position=cache.base_position)
    oc.k_chunks = cache.chunk_wire(unit, "k")[:n]
    oc.v_chunks = cache.chunk_wire(unit, "v")[:n]
    oc.k_res = np.zeros((0, 128), np.float32)
    oc.v_res = np.zeros((0, 128), np.float32)
    oc.total = n * 64
    return oc.attend(q_unit)[2]


def _attend_counts(cache, q, counts, no_lut):
    import torch

    from paper_2505_18231_b200 import _lib

    Hq = q.shape[1]
    cv = cache.view(Hq)
    n_chunks = torch.tensor(counts, dtype=torch.int32, device="cuda")
    n_res = torch.zeros(len(counts), dtype=torch.int32, device="cuda")
    cv.n_chunks = n_chunks.data_ptr()
    cv.n_res = n_res.data_ptr()
    cv.total_chunks = int(sum(counts))
    out = torch.full(tuple(q.shape), float("nan"), device="cuda")
    ws = cache._workspace(cv)
    old = os.environ.pop("NSNKV_NO_LUT", None)
    if no_lut:
        os.environ["NSNKV_NO_LUT"] = "1"
    try:
        _lib.check(_lib.lib.nsnkv_decode_attend(cv, q.data_ptr(), out.data_ptr(), None,
                                                ws.data_ptr(), ws.numel(),
                                                torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
    finally:
        os.environ.pop("NSNKV_NO_LUT", None)
        if old is not None:
            os.environ["NSNKV_NO_LUT"] = old
    return out.cpu().numpy()


def test_lut_ragged_units_vs_oracle():
    """512 units of 0..20 chunks (~5K chunks: every CTA steps through ~4
    units, some empty): every sampled unit matches the oracle, and the table
    path differs from the gather path only by rounding."""
    import torch

    import paper_2505_18231_b200 as P

    B, Hkv, G, T = 64, 8, 4, 64 * 20
    cb = P.default_codebook("1b")
    cfg = P.CacheConfig(d=128, bit_mode=cb.bit_mode)
    cache = P.PagedKvCache(cfg, B, Hkv, max_tokens=T, cb_k=cb, cb_v=cb, check_finite=False,
                           base_position=1000)  # RoPE positions offset (shift term)
    assert cache.precision == "vfast"
    g = torch.Generator(device="cuda")
    g.manual_seed(41)
    cache.append(torch.randn(B, Hkv, T, 128, device="cuda", generator=g),
                 torch.randn(B, Hkv, T, 128, device="cuda", generator=g))
    q = torch.randn(B, Hkv * G, 128, device="cuda", generator=g)
    rng = np.random.default_rng(7)
    counts = [int(c) for c in rng.integers(0, 21, size=B * Hkv)]
    for u in range(0, B * Hkv, 37):
        counts[u] = 0
    assert sum(counts) >= 32 * 148
    lut = _attend_counts(cache, q, counts, no_lut=False)
    gat = _attend_counts(cache, q, counts, no_lut=True)
    assert np.isfinite(lut).all() and np.isfinite(gat).all()
    qn = q.cpu().numpy()
    worst = 0.0
    for u in list(range(0, B * Hkv, 13)) + [B * Hkv - 1]:
        b, hk = divmod(u, Hkv)
        rows = lut[b, hk * G:(hk + 1) * G]
        if counts[u] == 0:
            assert np.all(rows == 0.0)
            continue
        ref = _oracle(cache, u, counts[u], qn[b, hk * G:(hk + 1) * G])
        for i in range(G):
            err = np.max(np.abs(rows[i] - ref[i])) / np.max(np.abs(ref[i]))
            worst = max(worst, err)
            assert err <= TOL, (u, counts[u], i, err)
    d = np.abs(lut - gat).max(axis=-1) / np.maximum(np.abs(gat).max(axis=-1), 1e-30)
    print(f"[lut ragged] worst vs oracle {worst:.2e}; table vs gather path {d.max():.2e}")
    assert d.max() <= 2e-4
    assert not np.array_equal(lut, gat)  # the two key paths really are different code


def test_lut_misaligned_vs_oracle():
    """Outlier data (verify.py:616-627 recipe) at 16K context, every unit:
    the fp32 table carries the key side at least as precisely as hi + lo."""
    import torch

    import paper_2505_18231_b200 as P
    from oracle import oracle as orc
    from tests.test_gpu_scale_parity import _misaligned_torch, _wire_all

    B, H, T, G = 4, 8, 16384, 4
    cb = P.default_codebook("1b")
    cfg = P.CacheConfig(d=128, bit_mode=cb.bit_mode)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(2026)
    cache = P.PagedKvCache(cfg, B, H, max_tokens=T, cb_k=cb, cb_v=cb, check_finite=False)
    cache.append(_misaligned_torch((B, H, T, 128), gen), _misaligned_torch((B, H, T, 128), gen))
    assert B * H * (T // 64) >= 32 * 148
    q = torch.randn(B, H * G, 128, device="cuda", generator=gen)
    out = cache.attend(q).cpu().numpy().reshape(B * H, G, 128)
    kw, vw = _wire_all(cache, "k"), _wire_all(cache, "v")
    ref = orc.attend_many(kw, vw, B * H, cache.n_chunks, cache.cb_k.entries, cache.cb_v.entries,
                          int(cache.bit_mode), q.cpu().numpy().reshape(B * H, G, 128))
    err = np.abs(out - ref).max(axis=-1) / np.abs(ref).max(axis=-1)
    print(f"[lut mis 16K] worst {err.max():.2e}, median {np.median(err):.2e}")
    assert err.max() <= TOL
