"""The packed cache as a model's attention backend (BASELINE config 5
conventions): one LLaMA-3.1-8B-shape layer (RoPE base 500000, GQA 32/8),
keys appended pre-RoPE and values in the Hadamard domain, q rotated at its
own position by the model; the fused serving step's attention output
matches the oracle (the reference restated) on the same pages within 1e-3."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "scripts"))

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", ["1b", "2b"])
def test_model_layer_attention_vs_oracle(mode):
    import bench_model as BM

    import paper_2505_18231_b200 as P
    from oracle import oracle as orc

    dev = torch.device("cuda", 0)
    model = BM.Model(1, dev, seed=3)
    L = model.layers[0]
    B, T = 2, 64 * 7 + 20
    cb = P.default_codebook(mode)
    cache = P.PagedKvCache(P.CacheConfig(d=128, bit_mode=cb.bit_mode, rope_base=BM.ROPE_BASE), B,
                           BM.N_KV, cb_k=cb, cb_v=cb)
    g = torch.Generator(device=dev)
    g.manual_seed(8)
    # prefill: the layer's own K/V projections of random hidden states
    hs = torch.randn(B, T, BM.D_MODEL, device=dev, generator=g).to(torch.bfloat16)
    qkv = (BM.rms_norm(hs, L["ln1"]) @ L["wqkv"]).float()
    k = qkv[..., BM.N_Q * 128:(BM.N_Q + BM.N_KV) * 128].view(B, T, BM.N_KV, 128).transpose(1, 2)
    v = qkv[..., (BM.N_Q + BM.N_KV) * 128:].view(B, T, BM.N_KV, 128).transpose(1, 2)
    cache.append(k.contiguous(), v.contiguous())
    # one decode step at position T
    h1 = torch.randn(B, BM.D_MODEL, device=dev, generator=g).to(torch.bfloat16)
    qkv1 = (BM.rms_norm(h1, L["ln1"]) @ L["wqkv"]).float()
    q = model.rope(qkv1[:, :BM.N_Q * 128].view(B, BM.N_Q, 128), T)
    k1 = qkv1[:, BM.N_Q * 128:(BM.N_Q + BM.N_KV) * 128].view(B, BM.N_KV, 1, 128)
    v1 = qkv1[:, (BM.N_Q + BM.N_KV) * 128:].view(B, BM.N_KV, 1, 128)
    out = cache.decode_step(q, k1.contiguous(), v1.contiguous()).cpu().numpy()
    G = BM.N_Q // BM.N_KV
    qn = q.cpu().numpy()
    worst = 0.0
    for u in range(B * BM.N_KV):
        b, hk = divmod(u, BM.N_KV)
        oc = orc.OracleCache(cb.entries, cb.entries, int(cb.bit_mode), rope_base=BM.ROPE_BASE)
        oc.k_chunks = cache.chunk_wire(u, "k")
        oc.v_chunks = cache.chunk_wire(u, "v")
        n = int(cache.unit_n_res[u])
        oc.k_res = cache.k_res[u, :n].cpu().numpy()
        oc.v_res = cache.v_res[u, :n].cpu().numpy()
        oc.total = int(cache.unit_total[u])
        _, _, ref = oc.attend(qn[b, hk * G:(hk + 1) * G])
        got = out[b, hk * G:(hk + 1) * G]
        err = float((np.abs(got - ref).max(axis=-1) / np.abs(ref).max(axis=-1)).max())
        worst = max(worst, err)
    print(f"[{mode}] model-layer attention worst rel err {worst:.2e}")
    assert worst <= 1e-3
