"""Cache semantics on the GPU (reference pkg/tests/test_kvcache.py:35-60,
verify.py:387-425): chunk boundaries depend only on the token stream, so a
decode-style token-by-token fill, ragged batches and one prefill produce
byte-identical caches; counters and residual bookkeeping follow the
reference policy."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _cache(mode="2b", B=2, H=2, base=0):
    import paper_2505_18231_b200 as P

    cb = P.default_codebook(mode)
    cfg = P.CacheConfig(d=128, bit_mode=cb.bit_mode)
    return P.PagedKvCache(cfg, B, H, cb_k=cb, cb_v=cb, base_position=base)


@pytest.mark.parametrize("mode", ["1b", "2b"])
def test_decode_fill_equals_prefill(mode):
    B, H, T = 2, 2, 64 * 3 + 7
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    k = torch.randn(B, H, T, 128, device="cuda", generator=g)
    v = torch.randn(B, H, T, 128, device="cuda", generator=g)
    pre = _cache(mode, B, H)
    pre.append(k, v)
    dec = _cache(mode, B, H)
    for i in range(T):  # one token per step, like a decode loop
        dec.append(k[:, :, i:i + 1], v[:, :, i:i + 1])
    rag = _cache(mode, B, H)
    for a, b in [(0, 5), (5, 64), (64, 65), (65, 190), (190, T)]:
        rag.append(k[:, :, a:b], v[:, :, a:b])
    for u in range(B * H):
        s = pre.snapshot(u)
        assert dec.snapshot(u) == s
        assert rag.snapshot(u) == s
    q = torch.randn(B, 4 * H, 128, device="cuda", generator=g)
    assert torch.equal(pre.attend(q), dec.attend(q))


def test_reserve_presizes_and_keeps_results():
    """reserve() sizes the pools once; appends up to the reserved length never
    reallocate, and the cache contents equal an unreserved cache's."""
    B, H, T = 2, 2, 64 * 5 + 3
    g = torch.Generator(device="cuda")
    g.manual_seed(4)
    k = torch.randn(B, H, T, 128, device="cuda", generator=g)
    v = torch.randn(B, H, T, 128, device="cuda", generator=g)
    a = _cache("2b", B, H).reserve(T)
    pools = (a.pool_ptrs(), a.capacity, a.max_chunks)
    b = _cache("2b", B, H)
    for i in range(0, T, 7):
        a.append(k[:, :, i:i + 7], v[:, :, i:i + 7])
        b.append(k[:, :, i:i + 7], v[:, :, i:i + 7])
    assert (a.pool_ptrs(), a.capacity, a.max_chunks) == pools
    for u in range(B * H):
        assert a.snapshot(u) == b.snapshot(u)
    q = torch.randn(B, 4 * H, 128, device="cuda", generator=g)
    assert torch.equal(a.attend(q), b.attend(q))


def test_chunk_counting_and_residual():
    # reference test_kvcache.py:35-50: 130 tokens -> 2 chunks + 2 residual rows
    c = _cache("2b", 1, 1)
    x = torch.randn(1, 1, 130, 128, device="cuda")
    c.append(x, x)
    assert c.n_chunks == 2 and c.n_res == 2 and c.total_tokens == 130
    assert torch.equal(c.k_res[0, :2], x[0, 0, 128:])


def test_base_position_enters_rotation():
    x = torch.randn(1, 1, 64, 128, device="cuda")
    a = _cache("2b", 1, 1, base=0)
    b = _cache("2b", 1, 1, base=1000)
    a.append(x, x)
    b.append(x, x)
    # values are not rotated, keys are
    assert a.pages(0, "v").tobytes() == b.pages(0, "v").tobytes()
    assert a.pages(0, "k").tobytes() != b.pages(0, "k").tobytes()


def test_bf16_input_equals_fp32_of_the_same_values():
    x = torch.randn(2, 2, 130, 128, device="cuda").to(torch.bfloat16)
    a = _cache("1b")
    b = _cache("1b")
    a.append(x, x)
    b.append(x.float(), x.float())
    for u in range(4):
        assert a.snapshot(u) == b.snapshot(u)


def test_rejects_non_finite_and_bad_shapes():
    from paper_2505_18231_b200 import ShapeMismatch

    c = _cache("2b", 1, 1)
    bad = torch.full((1, 1, 3, 128), float("nan"), device="cuda")
    with pytest.raises(ValueError):
        c.append(bad, bad)
    with pytest.raises(ShapeMismatch):
        c.append(torch.zeros(1, 1, 3, 64, device="cuda"), torch.zeros(1, 1, 3, 64, device="cuda"))
    with pytest.raises(ShapeMismatch):
        c.attend(torch.zeros(1, 4, 128, device="cuda"))  # empty cache


def test_sharded_decoder_single_rank_is_identity():
    from paper_2505_18231_b200.sharding import ShardedDecoder, plan_shards

    c = _cache("2b", 2, 2)
    x = torch.randn(2, 2, 100, 128, device="cuda")
    dec = ShardedDecoder(plan_shards(2, 2, 8, 1, 0), c)
    dec.append(x, x)
    q = torch.randn(2, 8, 128, device="cuda")
    assert torch.equal(dec.attend(q), c.attend(q))


def test_level1_api_snapshot_matches_batched():
    import paper_2505_18231_b200 as P

    cb = P.default_codebook("2b")
    cfg = P.CacheConfig(d=128, bit_mode="2b")
    st = P.new_cache(cfg)
    rng = np.random.default_rng(0)
    k = rng.standard_normal((150, 128)).astype(np.float32)
    v = rng.standard_normal((150, 128)).astype(np.float32)
    P.append(st, k, v, cb, cb)
    c = _cache("2b", 1, 1)
    c.append(torch.from_numpy(k)[None, None].cuda(), torch.from_numpy(v)[None, None].cuda())
    assert hashlib.sha256(P.snapshot(st)).hexdigest() == hashlib.sha256(c.snapshot(0)).hexdigest()
    assert st.n_chunks == 2 and st.residual_count == 22
    assert list(st.residual_positions) == list(range(128, 150))
