"""Fused decode (nsnkv_decode_attend) with ragged per-unit chunk counts,
driven through the C ABI: units with 0, 1, 2, ... chunks side by side, odd
counts (single-chunk work items), totals below the SM count (a grid of fewer
CTAs than SMs) and units spanning several CTAs (stream-K records).  Each unit's
output is checked against the oracle run on the unit's first n_u chunks
(reference attention.py:136-142).  Tolerance: max|d out| <= 1e-3 * max|out|
per (batch, q-head), the north-star bound."""

from __future__ import annotations

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


@pytest.mark.parametrize("mode,G,precision,counts", [
    ("2b", 4, "vfast", [0, 1, 2, 3, 9, 5, 0, 7, 1, 4, 8, 6]),
    ("2b", 4, "precise", [3, 0, 1, 9, 2, 2, 5, 0, 7, 1, 9, 4]),
    ("2b", 1, None, [1, 0, 0, 2, 3, 1, 5, 0, 1, 1, 2, 1]),   # 17 chunks: grid of 17 CTAs
    ("1b", 8, None, [9, 9, 9, 9, 9, 9, 9, 9, 9, 9, 9, 0]),
    ("1b", 2, None, [0, 0, 0, 0, 0, 1, 0, 0, 0, 0, 0, 0]),   # one chunk in the whole batch
])
def test_ragged_units_vs_oracle(mode, G, precision, counts):
    import torch

    import paper_2505_18231_b200 as P
    from paper_2505_18231_b200 import _lib

    B, Hkv, T = 3, 4, 64 * 9
    cb = P.default_codebook(mode)
    cfg = P.CacheConfig(d=128, bit_mode=cb.bit_mode)
    cache = P.PagedKvCache(cfg, B, Hkv, max_tokens=T, cb_k=cb, cb_v=cb, precision=precision)
    g = torch.Generator(device="cuda")
    g.manual_seed(sum(counts) + G)
    cache.append(torch.randn(B, Hkv, T, 128, device="cuda", generator=g),
                 torch.randn(B, Hkv, T, 128, device="cuda", generator=g))
    q = torch.randn(B, Hkv * G, 128, device="cuda", generator=g)
    cv = cache.view(Hkv * G)
    n_chunks = torch.tensor(counts, dtype=torch.int32, device="cuda")
    n_res = torch.zeros(B * Hkv, dtype=torch.int32, device="cuda")
    cv.n_chunks = n_chunks.data_ptr()
    cv.n_res = n_res.data_ptr()
    cv.total_chunks = int(sum(counts))
    out = torch.full((B, Hkv * G, 128), float("nan"), device="cuda")
    ws = cache._workspace(cv)
    _lib.check(_lib.lib.nsnkv_decode_attend(cv, q.data_ptr(), out.data_ptr(), None, ws.data_ptr(),
                                            ws.numel(), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    qn = q.cpu().numpy()
    for u, n in enumerate(counts):
        b, hk = divmod(u, Hkv)
        rows = got[b, hk * G:(hk + 1) * G]
        if n == 0:  # nothing cached for the unit: zero output, no NaN
            assert np.all(rows == 0.0)
            continue
        ref = _oracle(cache, u, n, qn[b, hk * G:(hk + 1) * G])
        for i in range(G):
            err = np.max(np.abs(rows[i] - ref[i]))
            assert err <= TOL * np.max(np.abs(ref[i])), (u, n, i, err)
