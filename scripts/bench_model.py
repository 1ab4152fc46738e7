"""Full-model decode step (BASELINE config 5): random-init LLaMA-3.1-8B
(32 layers, d_model 4096, 32 q / 8 KV heads of 128, SwiGLU 14336, RMSNorm,
RoPE base 500000, vocab 128256, bf16 weights) decoding one token per
sequence with

  --kv nsn1b / nsn2b : the NSNQuant packed cache (paper_2505_18231_b200) as
                       the attention backend -- the new K/V of every layer
                       are appended (a 64-token chunk is flushed through the
                       encode kernel every 64 steps) and attention runs the
                       fused packed-KV decode kernel;
  --kv bf16          : a bf16 KV cache with flash-attn's decode kernel
                       (flash_attn_with_kvcache), the usual serving baseline.

The dense parts (projections, MLP, lm_head) are plain torch/cuBLAS bf16 in
both arms, so the difference is the KV cache.  The value projection is taken
to emit Hadamard-domain values (the reference's fused-projection convention,
kvcache.py:138-154); with random weights this is a relabelling.  Prints one
JSON line.
"""

from __future__ import annotations

import argparse
import json
import math
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

D_MODEL, N_Q, N_KV, HD, FFN, VOCAB = 4096, 32, 8, 128, 14336, 128256
ROPE_BASE = 500000.0


def rms_norm(x, w, eps=1e-5):
    xf = x.float()
    return (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + eps)).to(x.dtype) * w


class Model:
    def __init__(self, n_layers, dev, seed=0):
        g = torch.Generator(device=dev)
        g.manual_seed(seed)

        def w(*shape, scale):
            return (torch.randn(*shape, device=dev, generator=g) * scale).to(torch.bfloat16)

        self.layers = []
        for _ in range(n_layers):
            self.layers.append({
                "ln1": torch.ones(D_MODEL, device=dev, dtype=torch.bfloat16),
                "wqkv": w(D_MODEL, (N_Q + 2 * N_KV) * HD, scale=D_MODEL ** -0.5),
                "wo": w(N_Q * HD, D_MODEL, scale=(N_Q * HD) ** -0.5),
                "ln2": torch.ones(D_MODEL, device=dev, dtype=torch.bfloat16),
                "wgu": w(D_MODEL, 2 * FFN, scale=D_MODEL ** -0.5),
                "wd": w(FFN, D_MODEL, scale=FFN ** -0.5),
            })
        self.emb = w(VOCAB, D_MODEL, scale=1.0)
        self.lnf = torch.ones(D_MODEL, device=dev, dtype=torch.bfloat16)
        self.head = w(D_MODEL, VOCAB, scale=D_MODEL ** -0.5)
        j = torch.arange(HD // 2, device=dev, dtype=torch.float64)
        self.freqs = ROPE_BASE ** (-2.0 * j / HD)

    def rope(self, x, pos):
        """Rotate [..., 128] fp32 at one position (pairs 2j, 2j+1)."""
        th = pos * self.freqs
        c, s = torch.cos(th).float(), torch.sin(th).float()
        e, o = x[..., 0::2], x[..., 1::2]
        out = torch.empty_like(x)
        out[..., 0::2] = e * c - o * s
        out[..., 1::2] = e * s + o * c
        return out


def build_nsn(model, args, dev, bit_mode):
    import paper_2505_18231_b200 as P

    cb = P.default_codebook(f"{bit_mode}b")
    cfg = P.CacheConfig(d=HD, bit_mode=cb.bit_mode, rope_base=ROPE_BASE)
    caches = []
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    for _ in model.layers:
        c = P.PagedKvCache(cfg, args.batch, N_KV, max_tokens=args.context + args.steps + 64,
                           cb_k=cb, cb_v=cb, device=dev, check_finite=False,
                           precision=args.precision)
        done = 0
        while done < args.context:
            n = min(2048, args.context - done)
            c.append(torch.randn(args.batch, N_KV, n, HD, device=dev, generator=g).to(torch.bfloat16),
                     torch.randn(args.batch, N_KV, n, HD, device=dev, generator=g).to(torch.bfloat16))
            done += n
        caches.append(c)
    torch.cuda.synchronize()
    return caches


def build_bf16(model, args, dev):
    caches = []
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    cap = args.context + args.steps + 64
    for _ in model.layers:
        k = torch.empty(args.batch, cap, N_KV, HD, device=dev, dtype=torch.bfloat16)
        v = torch.empty_like(k)
        k[:, :args.context].normal_(generator=g)
        v[:, :args.context].normal_(generator=g)
        caches.append((k, v))
    torch.cuda.synchronize()
    return caches


def step(model, caches, x_tok, pos, kind):
    B = x_tok.shape[0]
    x = model.emb[x_tok]
    for li, L in enumerate(model.layers):
        h = rms_norm(x, L["ln1"])
        qkv = h @ L["wqkv"]
        q = qkv[:, :N_Q * HD].view(B, N_Q, HD).float()
        k = qkv[:, N_Q * HD:(N_Q + N_KV) * HD].view(B, N_KV, HD)
        v = qkv[:, (N_Q + N_KV) * HD:].view(B, N_KV, HD)
        q = model.rope(q, pos)
        if kind == "bf16":
            from flash_attn import flash_attn_with_kvcache

            kc, vc = caches[li]
            k_r = model.rope(k.float(), pos).to(torch.bfloat16)
            seqlens = torch.full((B,), pos, dtype=torch.int32, device=x.device)
            o = flash_attn_with_kvcache(q.to(torch.bfloat16)[:, None], kc, vc, k=k_r[:, None],
                                        v=v[:, None], cache_seqlens=seqlens, causal=True)
            o = o.view(B, N_Q * HD)
        else:
            # keys pre-RoPE, values HT-domain: one fused serving step (the new
            # token is attended and stored by the attend launches; a chunk is
            # flushed through nsnkv_append every 64 steps)
            o = caches[li].decode_step(q, k[:, :, None], v[:, :, None]).to(torch.bfloat16)
            o = o.view(B, N_Q * HD)
        x = x + o @ L["wo"]
        h = rms_norm(x, L["ln2"])
        gu = h @ L["wgu"]
        x = x + (torch.nn.functional.silu(gu[:, :FFN]) * gu[:, FFN:]) @ L["wd"]
    logits = rms_norm(x, model.lnf) @ model.head
    return logits.argmax(-1)


def run(kv: str, batch: int, context: int, layers: int, steps: int, warmup: int, dev,
        precision: str | None = None, dp: int = 8) -> dict:
    """One arm of BASELINE config 5 on one GPU: batch sequences (the per-GPU
    share of a data-parallel job of dp replicas) at `context` tokens."""
    args = argparse.Namespace(kv=kv, batch=batch, context=context, layers=layers, steps=steps,
                              warmup=warmup, precision=precision)
    t0 = time.time()
    model = Model(args.layers, dev)
    if args.kv == "bf16":
        caches = build_bf16(model, args, dev)
        kv_bytes = sum(k.numel() * 2 * 2 for k, _ in caches) * args.context // (args.context + args.steps + 64)
    else:
        caches = build_nsn(model, args, dev, 1 if args.kv == "nsn1b" else 2)
        ledger = 1268 if args.kv == "nsn1b" else 2292
        kv_bytes = args.layers * args.batch * N_KV * (args.context // 64) * ledger * 2
    build_s = time.time() - t0
    tok = torch.zeros(args.batch, dtype=torch.long, device=dev)
    pos = args.context
    for _ in range(args.warmup):
        tok = step(model, caches, tok, pos, args.kv)
        pos += 1
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        tok = step(model, caches, tok, pos, args.kv)
        pos += 1
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    res = {
        "metric": "full-model decode step", "kv": args.kv, "model": "LLaMA-3.1-8B shape, random init",
        "batch_per_gpu": args.batch, "context": args.context, "layers": args.layers,
        "ms_per_step": round(ms, 3), "tokens_per_s_per_gpu": round(args.batch / (ms * 1e-3), 1),
        "dp": dp, "global_batch": dp * args.batch,
        "tokens_per_s_job": round(dp * args.batch / (ms * 1e-3), 1),
        "kv_cache_GB_per_gpu": round(kv_bytes / 1e9, 2),
        "max_mem_GB": round(torch.cuda.max_memory_allocated() / 1e9, 1),
        "build_s": round(build_s, 1), "precision": (caches[0].precision if args.kv != "bf16" else "bf16"),
        "how": f"one GPU measured; the data-parallel job is {dp} independent replicas (decode needs no "
               f"cross-replica exchange), so job tokens/s = {dp} x per-GPU",
    }
    del caches, model
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kv", default="nsn1b", choices=["nsn1b", "nsn2b", "bf16"])
    ap.add_argument("--batch", type=int, default=32, help="sequences per GPU (C5: 256 / DP 8)")
    ap.add_argument("--context", type=int, default=16384)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--dp", type=int, default=8)
    ap.add_argument("--precision", default=None)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    print(json.dumps(run(args.kv, args.batch, args.context, args.layers, args.steps, args.warmup,
                         dev, args.precision, args.dp)), flush=True)


if __name__ == "__main__":
    main()
