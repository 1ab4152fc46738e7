"""Randomised appends against the oracle, bit for bit: bit mode, scale
strategy, fp32 or bf16 input, N(0,1) or misaligned (outlier) rows, RoPE base
position and a sequence of ragged appends (per-sequence lengths through
``seq_lens``, residual carry-over included) are drawn from a fixed seed.
Every unit's chunks, converted to the reference wire format, must equal the
chunks the oracle's restatement of kvcache.append (kvcache.py:157-195) makes
from the same rows, and the residual rows must match."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _misaligned(rng, n):
    from tests.golden.inputs import misaligned

    return misaligned(rng, n)


def _cases(n=10, seed=77):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        out.append(dict(i=i, mode="1b" if rng.random() < 0.5 else "2b",
                        strategy=int(rng.integers(0, 4)), bf16=bool(rng.random() < 0.5),
                        mis=bool(rng.random() < 0.5), B=int(rng.integers(1, 5)),
                        H=int(rng.choice([1, 2, 8])), base=int(rng.choice([0, 5, 1000])),
                        steps=int(rng.integers(2, 5))))
    return out


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"e{c['i']}-{c['mode']}-s{c['strategy']}")
def test_random_appends_vs_oracle(case):
    import torch

    import paper_2505_18231_b200 as P
    from oracle import oracle as orc

    rng = np.random.default_rng(500 + case["i"])
    cb = P.default_codebook(case["mode"])
    cfg = P.CacheConfig(d=128, bit_mode=cb.bit_mode, strategy=P.ScaleStrategy(case["strategy"]))
    B, H = case["B"], case["H"]
    cache = P.PagedKvCache(cfg, B, H, cb_k=cb, cb_v=cb, base_position=case["base"],
                           check_finite=False)
    refs = [orc.OracleCache(cb.entries, cb.entries, int(cb.bit_mode), strategy=case["strategy"],
                            base_position=case["base"]) for _ in range(B * H)]
    for step in range(case["steps"]):
        lens = [int(x) for x in rng.integers(0, 150, size=B)]
        if sum(lens) == 0:
            lens[0] = 1
        tot = sum(lens)
        gen = (lambda n: _misaligned(rng, n)) if case["mis"] else (
            lambda n: rng.standard_normal((n, 128)).astype(np.float32))
        K = np.stack([gen(tot) for _ in range(H)], axis=1)  # [tot, H, 128]
        V = np.stack([gen(tot) for _ in range(H)], axis=1)
        if case["bf16"]:  # both sides see the same bf16-rounded values
            K = torch.from_numpy(K).bfloat16().float().numpy()
            V = torch.from_numpy(V).bfloat16().float().numpy()
        kt = torch.from_numpy(K).cuda()
        vt = torch.from_numpy(V).cuda()
        if case["bf16"]:
            kt, vt = kt.bfloat16(), vt.bfloat16()
        cache.append(kt, vt, seq_lens=lens)
        off = 0
        for b in range(B):
            for h in range(H):
                if lens[b]:
                    refs[b * H + h].append(K[off:off + lens[b], h], V[off:off + lens[b], h])
            off += lens[b]
    torch.cuda.synchronize()
    for u, ref in enumerate(refs):
        assert cache.chunk_wire(u, "k") == ref.k_chunks, (case, u, "k")
        assert cache.chunk_wire(u, "v") == ref.v_chunks, (case, u, "v")
        n_res = ref.k_res.shape[0]
        assert int(cache.unit_n_res[u]) == n_res
        if n_res:
            assert np.array_equal(cache.k_res[u, :n_res].cpu().numpy(), ref.k_res)
            assert np.array_equal(cache.v_res[u, :n_res].cpu().numpy(), ref.v_res)
