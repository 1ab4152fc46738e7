"""Randomised decode configurations against the oracle: bit mode, GQA group,
precision mode, batch / head counts, context lengths,
RoPE base positions and per-unit chunk counts (ragged through the C ABI) are
drawn from a fixed seed, sized so that CTAs run several work items and, for
1-bit G = 4, the key-table path is taken.  Each case checks a sample of units
(every empty unit must return zeros).  Tolerance: max|d out| <= 1e-3 *
max|out| per (batch, q-head), reference attention.py:136-142 restated by the
oracle on the GPU's own pages."""

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


def _cases(n=14, seed=2027):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        mode = "1b" if rng.random() < 0.5 else "2b"
        G = int(rng.choice([1, 2, 4, 8]))
        prec = str(rng.choice(["vfast", "precise"]))
        Hkv = int(rng.choice([2, 4, 8]))
        B = int(rng.integers(2, 9))
        nch = int(rng.integers(8, 90))
        base = int(rng.choice([0, 0, 17, 4096]))
        out.append((i, mode, G, prec, B, Hkv, nch, base))
    # one case certain to take the 1-bit key-table path (>= 32 chunks per CTA)
    out.append((n, "1b", 4, "vfast", 8, 8, 160, 300))
    return out


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"c{c[0]}-{c[1]}-G{c[2]}-{c[3]}")
def test_random_decode_vs_oracle(case):
    import torch

    import paper_2505_18231_b200 as P
    from paper_2505_18231_b200 import _lib

    i, mode, G, prec, B, Hkv, nch, base = case
    cb = P.default_codebook(mode)
    cfg = P.CacheConfig(d=128, bit_mode=cb.bit_mode)
    T = 64 * nch
    cache = P.PagedKvCache(cfg, B, Hkv, max_tokens=T, cb_k=cb, cb_v=cb, precision=prec,
                           base_position=base, check_finite=False)
    g = torch.Generator(device="cuda")
    g.manual_seed(1000 + i)
    cache.append(torch.randn(B, Hkv, T, 128, device="cuda", generator=g),
                 torch.randn(B, Hkv, T, 128, device="cuda", generator=g))
    q = torch.randn(B, Hkv * G, 128, device="cuda", generator=g)
    rng = np.random.default_rng(i)
    units = B * Hkv
    lo = nch // 2 if nch >= 160 else 0
    counts = [int(c) for c in rng.integers(lo, nch + 1, size=units)]
    counts[0] = 0              # an empty unit
    counts[units - 1] = nch    # a full one
    cv = cache.view(Hkv * G)
    n_chunks = torch.tensor(counts, dtype=torch.int32, device="cuda")
    n_res = torch.zeros(units, dtype=torch.int32, device="cuda")
    cv.n_chunks = n_chunks.data_ptr()
    cv.n_res = n_res.data_ptr()
    cv.total_chunks = int(sum(counts))
    out = torch.full((B, Hkv * G, 128), float("nan"), device="cuda")
    ws = cache._workspace(cv)
    _lib.check(_lib.lib.nsnkv_decode_attend(cv, q.data_ptr(), out.data_ptr(), None, ws.data_ptr(),
                                            ws.numel(), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    assert np.isfinite(got).all()
    qn = q.cpu().numpy()
    sample = sorted(set(rng.choice(units, size=min(units, 10), replace=False).tolist()
                        + [0, units - 1]))
    worst = 0.0
    for u in sample:
        b, hk = divmod(u, Hkv)
        rows = got[b, hk * G:(hk + 1) * G]
        if counts[u] == 0:
            assert np.all(rows == 0.0), u
            continue
        ref = _oracle(cache, u, counts[u], qn[b, hk * G:(hk + 1) * G])
        for h in range(G):
            err = np.max(np.abs(rows[h] - ref[h])) / np.max(np.abs(ref[h]))
            worst = max(worst, err)
            assert err <= TOL, (case, u, counts[u], h, err)
    print(f"[fuzz {case}] {sum(counts)} chunks, worst {worst:.2e}")
