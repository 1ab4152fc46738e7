"""Parity at BASELINE scale, GPU against the oracle (the reference restated
operation by operation, pinned to the reference's goldens in
test_oracle_golden.py / test_c1_parity.py):

  * encode at C3 scale (16,384 chunks per side, bf16 activations like C3):
    every page bit-identical to the oracle's serialized chunk, counters equal;
  * decode at C2 scale (B16 x 8 KV heads x 32K, GQA 4): EVERY one of the 128
    units' 4 q-heads within 1e-3, in both 2-bit precision modes, and a
    misaligned-data C2-shaped case (large-magnitude outlier scores, where a
    plain-fp16 key codeword breaks the tolerance).
"""

from __future__ import annotations

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-3
THREADS = os.cpu_count() or 8


def _misaligned_torch(shape, gen):
    """tests/golden/inputs.misaligned on the GPU: channel-scale outliers,
    nonzero channel means, 1 % of tokens scaled by 50."""
    import torch

    x = torch.randn(*shape, device="cuda", generator=gen)
    scales = torch.ones(128, device="cuda")
    scales[::16] = 10.0
    means = torch.zeros(128, device="cuda")
    means[::8] = 2.0
    x = x * scales + means
    hit = torch.rand(*shape[:-1], device="cuda", generator=gen) < 0.01
    return torch.where(hit[..., None], x * 50.0, x)


def _wire_all(cache, kind):
    from paper_2505_18231_b200.cache import pages_to_wire

    return pages_to_wire(cache.all_pages(kind), cache.bit_mode, cache.config.strategy, kind)


@pytest.mark.parametrize("mode,dist,B,T", [("2b", "normal", 8, 16384), ("1b", "mis", 8, 16384),
                                            # BASELINE config 3 at full size: 65,536 chunks per side
                                            ("2b", "normal", 64, 8192), ("1b", "normal", 64, 8192)])
def test_encode_c3_scale_bit_exact_vs_oracle(mode, dist, B, T):
    import torch

    import paper_2505_18231_b200 as P
    from oracle import oracle as orc

    H = 8
    cb = P.default_codebook(mode)
    cfg = P.CacheConfig(d=128, bit_mode=cb.bit_mode)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(77)
    if dist == "normal":
        k = torch.randn(B, H, T, 128, device="cuda", generator=gen)
        v = torch.randn(B, H, T, 128, device="cuda", generator=gen)
    else:
        k = _misaligned_torch((B, H, T, 128), gen)
        v = _misaligned_torch((B, H, T, 128), gen)
    k, v = k.bfloat16(), v.bfloat16()
    cache = P.PagedKvCache(cfg, B, H, max_tokens=T, cb_k=cb, cb_v=cb, check_finite=False)
    cache.append(k, v)
    n = B * H * (T // 64)
    pos0 = np.tile(np.arange(T // 64, dtype=np.int64) * 64, B * H)
    for kind, x in (("k", k), ("v", v)):
        rows = x.float().reshape(n, 64, 128).cpu().numpy()
        ref = orc.encode_many_pos(rows, kind == "k", pos0, cb.entries, int(cb.bit_mode),
                                  threads=THREADS)
        got = _wire_all(cache, kind)
        bad = np.nonzero((got != ref).any(axis=1))[0]
        assert bad.size == 0, f"{kind}: {bad.size} of {n} chunks differ (first {bad[:5]})"
    print(f"[{mode} {dist}] {n} chunks per side bit-exact; near-ties re-scored "
          f"{int(cache.counters()[:, 3].sum())}")


@pytest.fixture(scope="module")
def c2_cache():
    import torch

    import paper_2505_18231_b200 as P

    B, H, T = 16, 8, 32768
    cb = P.default_codebook("2b")
    cfg = P.CacheConfig(d=128, bit_mode=cb.bit_mode)
    cache = P.PagedKvCache(cfg, B, H, max_tokens=T, cb_k=cb, cb_v=cb, check_finite=False)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(2024)
    for t0 in range(0, T, 4096):
        cache.append(torch.randn(B, H, 4096, 128, device="cuda", generator=gen).bfloat16(),
                     torch.randn(B, H, 4096, 128, device="cuda", generator=gen).bfloat16())
    q = torch.randn(B, 32, 128, device="cuda", generator=gen)
    return cache, q


def _all_units_err(cache, q):
    from oracle import oracle as orc

    B, Hq = q.shape[:2]
    U = cache.units
    G = Hq // cache.n_kv_heads
    out = cache.attend(q).cpu().numpy().reshape(U, G, 128)
    kw = _wire_all(cache, "k")
    vw = _wire_all(cache, "v")
    ref = orc.attend_many(kw, vw, U, cache.n_chunks, cache.cb_k.entries, cache.cb_v.entries,
                          int(cache.bit_mode), q.cpu().numpy().reshape(U, G, 128), threads=THREADS)
    err = np.abs(out - ref).max(axis=-1) / np.abs(ref).max(axis=-1)
    return err


@pytest.mark.parametrize("precision", ["vfast", "precise"])
def test_decode_c2_all_units_vs_oracle(c2_cache, precision):
    cache, q = c2_cache
    cache.precision = precision
    err = _all_units_err(cache, q)
    print(f"[C2 {precision}] 128 units x 4 heads: worst {err.max():.2e}, median {np.median(err):.2e}")
    assert err.max() <= TOL, (precision, err.max(), np.unravel_index(err.argmax(), err.shape))


@pytest.mark.parametrize("mode,precision", [("2b", "vfast"), ("2b", "precise"), ("1b", "precise"),
                                            ("1b", "vfast")])
def test_decode_misaligned_long_context_vs_oracle(mode, precision):
    """Outlier tokens make scores large, so every relative error on a score
    is amplified by the softmax: the key codewords must carry ~22 bits
    (hi + lo).  A plain-fp16 key side fails this case."""
    import torch

    import paper_2505_18231_b200 as P

    B, H, T = 2, 8, 4096
    cb = P.default_codebook(mode)
    cfg = P.CacheConfig(d=128, bit_mode=cb.bit_mode)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(606)
    cache = P.PagedKvCache(cfg, B, H, max_tokens=T, cb_k=cb, cb_v=cb, check_finite=False,
                           precision=precision)
    cache.append(_misaligned_torch((B, H, T, 128), gen), _misaligned_torch((B, H, T, 128), gen))
    q = torch.randn(B, 32, 128, device="cuda", generator=gen)
    err = _all_units_err(cache, q)
    print(f"[mis {mode} {precision}] worst {err.max():.2e}")
    assert err.max() <= TOL
