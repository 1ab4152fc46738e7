"""Encode (prefill quantize + append) throughput, BASELINE config 3:
LLaMA-3.1-8B KV shape, batch 64 x 8K tokens x 8 KV heads, bf16 K/V in,
1-bit and 2-bit.  Prints one JSON line per bit mode.

bytes per launch (algorithmic) = K+V input read (bf16, 256 B per token-head
each) + packed pages written (ledger bytes).  The kernel is bound by the
codebook search (32,768 fp32 MAC per token vector), not by HBM.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2505_18231_b200 as P  # noqa: E402

LEDGER = {1: 1268, 2: 2292}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--heads", type=int, default=8)
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--modes", default="1,2")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    B, H, T = args.batch, args.heads, args.tokens
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    k = torch.randn(B, H, T, 128, device=dev, generator=g).to(torch.bfloat16)
    v = torch.randn(B, H, T, 128, device=dev, generator=g).to(torch.bfloat16)
    for mode in [int(m) for m in args.modes.split(",")]:
        cb = P.default_codebook(f"{mode}b")
        cfg = P.CacheConfig(d=128, bit_mode=cb.bit_mode)
        times = []
        launches = 0
        for it in range(args.steps + 1):
            cache = P.PagedKvCache(cfg, B, H, max_tokens=T, cb_k=cb, cb_v=cb, device=dev,
                                   check_finite=False)
            torch.cuda.synchronize()
            l0 = P._lib.launch_count()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            cache.append(k, v)
            e1.record()
            torch.cuda.synchronize()
            if it:  # first iteration is warm-up
                times.append(e0.elapsed_time(e1))
                launches = P._lib.launch_count() - l0
        ms = min(times)
        token_heads = B * H * T
        chunks = token_heads // 64
        nbytes = token_heads * 128 * 2 * 2 + chunks * LEDGER[mode] * 2
        cnt = cache.counters().sum(axis=0)
        print(json.dumps({
            "metric": "prefill encode throughput", "bit_mode": mode,
            "config": f"batch {B} x {H} kv-heads x {T} tokens, bf16 K/V in",
            "ms": round(ms, 3), "token_heads_per_s": round(token_heads / (ms * 1e-3), 1),
            "GBps_algorithmic": round(nbytes / (ms * 1e-3) / 1e9, 1),
            "match_TMACps": round(token_heads * 2 * 16 * 256 * 8 / (ms * 1e-3) / 1e12, 2),
            "gpu_launches": int(launches),
            "near_tie_subvectors": int(cnt[3]), "zero_subvectors": int(cnt[1]),
            "clamps": int(cnt[0]), "s3_fallbacks": int(cnt[2]),
        }), flush=True)


if __name__ == "__main__":
    main()
