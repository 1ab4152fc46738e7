"""GPU decode at BASELINE sizes: the fused kernel against the oracle on sampled
(batch, kv-head) units of the headline workload, plus size-independent
properties.  Tolerance: max|d out| <= 1e-3 * max|out| per (batch, q-head).
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-3


def _oracle_unit_out(cache, unit, q_unit):
    """Oracle decode of one unit from the GPU's own pages (converted to the
    reference wire format) and residual rows."""
    from oracle import oracle as orc

    cb = cache.cb_k
    oc = orc.OracleCache(cache.cb_k.entries, cache.cb_v.entries, int(cb.bit_mode),
                         base_position=cache.base_position)
    oc.k_chunks = cache.chunk_wire(unit, "k")
    oc.v_chunks = cache.chunk_wire(unit, "v")
    oc.k_res = cache.k_res[unit, :cache.n_res].cpu().numpy()
    oc.v_res = cache.v_res[unit, :cache.n_res].cpu().numpy()
    oc.total = cache.total_tokens
    _, _, out = oc.attend(q_unit)
    return out


def _build(B, Hkv, T, mode, seed, append_block=4096, precision="precise"):
    import torch

    import paper_2505_18231_b200 as P

    cb = P.default_codebook(mode)
    cfg = P.CacheConfig(d=128, bit_mode=cb.bit_mode)
    cache = P.PagedKvCache(cfg, B, Hkv, max_tokens=T, cb_k=cb, cb_v=cb, check_finite=False,
                           precision=precision, allow_inexact=precision == "fast")
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    done = 0
    while done < T:
        n = min(append_block, T - done)
        cache.append(torch.randn(B, Hkv, n, 128, device="cuda", generator=gen),
                     torch.randn(B, Hkv, n, 128, device="cuda", generator=gen))
        done += n
    return cache


@pytest.mark.parametrize("mode,B,Hq,Hkv,T,precision", [
    ("2b", 16, 32, 8, 32768, "vfast"),      # BASELINE config 2 (headline, default mode)
    ("2b", 4, 32, 8, 32768, "precise"),
    ("1b", 4, 32, 8, 32768 + 37, "precise"),  # 1-bit with a residual tail
    ("1b", 4, 32, 8, 32768 + 37, "vfast"),    # 1-bit default: fp16 values + mean-error term
    ("2b", 2, 8, 8, 4096 + 5, "vfast"),     # G = 1 (config 1 geometry)
    ("1b", 1, 8, 8, 4096, "precise"),       # config 1 itself
    ("1b", 1, 8, 8, 4096, "vfast"),
    ("2b", 3, 16, 2, 1000, "vfast"),        # G = 8, ragged
    ("2b", 2, 64, 8, 4096 + 5, "vfast"),    # G = 8, several work items per CTA (one-chunk items)
    ("1b", 2, 64, 8, 4096 + 5, "vfast"),
    ("2b", 2, 64, 8, 4096 + 5, "precise"),
    ("2b", 3, 16, 2, 1000, "precise"),
    ("1b", 2, 4, 2, 64 * 3, "precise"),     # G = 2
    ("1b", 2, 16, 8, 4096 + 5, "vfast"),    # G = 2, several work items per CTA
    ("2b", 2, 16, 8, 4096 + 5, "precise"),
    ("2b", 4, 32, 8, 8192 + 3, "fast"),     # opt-in fp16 mode (N(0,1) data), paired items
    ("1b", 2, 4, 2, 64 * 3, "vfast"),
    ("1b", 3, 16, 2, 1000, "vfast"),        # G = 8, 1-bit
])
def test_fused_decode_vs_oracle(mode, B, Hq, Hkv, T, precision):
    import torch

    cache = _build(B, Hkv, T, mode, seed=T + B, precision=precision)
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    q = torch.randn(B, Hq, 128, device="cuda", generator=g)
    out = cache.attend(q).cpu().numpy()
    qn = q.cpu().numpy()
    G = Hq // Hkv
    units = [0, B * Hkv - 1] if B * Hkv > 1 else [0]
    if B * Hkv > 4:
        units.append((B * Hkv) // 2 + 1)
    worst = 0.0
    for u in units:
        b, h = divmod(u, Hkv)
        ref = _oracle_unit_out(cache, u, qn[b, h * G:(h + 1) * G])
        got = out[b, h * G:(h + 1) * G]
        for i in range(G):
            err = np.max(np.abs(got[i] - ref[i])) / np.max(np.abs(ref[i]))
            worst = max(worst, err)
            assert err <= TOL, f"unit {u} head {i}: rel err {err:.2e}"
    print(f"[{mode} {precision} T={T} G={G}] worst max-rel error {worst:.2e}")
    assert np.isfinite(out).all()


def test_fused_decode_matches_unfused_path():
    """The fused kernel and the reference-shaped scores -> softmax -> output
    path agree on every (batch, q-head) of a mid-size cache."""
    import torch

    cache = _build(4, 4, 64 * 40 + 11, "2b", seed=3)
    q = torch.randn(4, 16, 128, device="cuda")
    fused = cache.attend(q)
    s = cache.scores(q).double() / np.sqrt(128.0)
    w = torch.softmax(s, dim=-1).float()
    unfused = cache.output(w)
    err = ((fused - unfused).abs().amax(dim=-1) / unfused.abs().amax(dim=-1)).max().item()
    assert err <= TOL


@pytest.mark.parametrize("mode,B,Hq,Hkv,T,precision", [
    ("2b", 2, 32, 8, 4096, "precise"),
    ("2b", 4, 32, 8, 16384 + 7, "vfast"),  # multi-item CTAs, stream-K merges
    ("1b", 8, 32, 8, 8192, "vfast"),       # key-table path
    ("2b", 2, 64, 8, 4096 + 5, "vfast"),   # GQA-8 (two-group CTA)
])
def test_decode_is_deterministic(mode, B, Hq, Hkv, T, precision):
    """Fixed merge orders everywhere (warps of a group, stream-K records, the
    combine): repeated decodes of the same cache are bit-identical."""
    import torch

    cache = _build(B, Hkv, T, mode, seed=9, precision=precision)
    q = torch.randn(B, Hq, 128, device="cuda")
    a = cache.attend(q).clone()
    for _ in range(10):
        assert torch.equal(a, cache.attend(q))


def test_decode_c4_full_size_vs_oracle():
    """BASELINE config 4 at full size on one GPU (batch 128 x 8 KV heads x
    128K tokens, 2-bit, 32 q-heads per sequence: 9.6 GB of pages): sampled
    units, first / middle / last, against the oracle on the GPU's own pages."""
    import torch

    B, Hq, Hkv, T = 128, 32, 8, 131072
    cache = _build(B, Hkv, T, "2b", seed=44, append_block=2048, precision="vfast")
    g = torch.Generator(device="cuda")
    g.manual_seed(45)
    q = torch.randn(B, Hq, 128, device="cuda", generator=g)
    out = cache.attend(q).cpu().numpy()
    qn = q.cpu().numpy()
    G = Hq // Hkv
    worst = 0.0
    for u in (0, (B * Hkv) // 2 + 3, B * Hkv - 1):
        b, h = divmod(u, Hkv)
        ref = _oracle_unit_out(cache, u, qn[b, h * G:(h + 1) * G])
        got = out[b, h * G:(h + 1) * G]
        for i in range(G):
            err = np.max(np.abs(got[i] - ref[i])) / np.max(np.abs(ref[i]))
            worst = max(worst, err)
            assert err <= TOL, (u, i, err)
    print(f"[C4 full size] worst max-rel error {worst:.2e}")
    assert np.isfinite(out).all()
