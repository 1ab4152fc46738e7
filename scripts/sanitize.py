"""Small end-to-end run for compute-sanitizer (memcheck / racecheck /
synccheck): ragged appends (nsnkv_append), fused decode (attend3 + combine),
the fused serving step (nsnkv_decode_step), unfused decode, snapshot import,
the 1-bit key-table decode, the codebook-build passes and the level-1 kernels."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2505_18231_b200 as P  # noqa: E402
from paper_2505_18231_b200 import codebook_build as CB  # noqa: E402
from paper_2505_18231_b200 import kernels  # noqa: E402

for mode, G, prec in (("2b", 4, "vfast"), ("2b", 4, "precise"), ("1b", 1, None), ("2b", 8, None)):
    cb = P.default_codebook(mode)
    cfg = P.CacheConfig(d=128, bit_mode=cb.bit_mode)
    B, H, T = 2, 2, 64 * 5 + 9
    c = P.PagedKvCache(cfg, B, H, cb_k=cb, cb_v=cb, precision=prec)
    x = torch.randn(B, H, T, 128, device="cuda")
    c.append(x, x)
    rows = torch.randn(70 + 3, H, 128, device="cuda")
    c.append(rows, rows, seq_lens=[70, 3])            # ragged: one unit pair flushes
    q = torch.randn(B, H * G, 128, device="cuda")
    out = c.attend(q)
    s = c.scores(q)
    w = torch.softmax(s.double() / 128 ** 0.5, -1).float()
    out2 = c.output(w) if c.unit_total.min() == c.unit_total.max() else out
    for _ in range(3):                                # fused serving steps
        tok = torch.randn(B, H, 1, 128, device="cuda")
        c.decode_step(q, tok, tok)
    d = P.PagedKvCache(cfg, B, H, cb_k=cb, cb_v=cb, precision=prec)
    d.load_snapshot(1, c.snapshot(0))
    d.attend(q)
    torch.cuda.synchronize()
    print(mode, G, c.precision, float((out - out2).abs().max()))
# multi-item CTAs (~13 chunks per CTA: several work items per consumer group,
# producers reusing their shift-term operand) in every gather-path mode,
# with fused serving steps
for mode, G, prec in (("2b", 4, "vfast"), ("2b", 4, "precise"), ("1b", 4, "precise"),
                      ("2b", 8, "vfast"), ("1b", 2, "vfast"), ("2b", 1, "vfast")):
    cb = P.default_codebook(mode)
    cfg = P.CacheConfig(d=128, bit_mode=cb.bit_mode)
    B, H, T = 4, 8, 64 * 60 + 5
    c = P.PagedKvCache(cfg, B, H, max_tokens=T + 8, cb_k=cb, cb_v=cb, precision=prec,
                       check_finite=False)
    x = torch.randn(B, H, T, 128, device="cuda")
    c.append(x, x)
    q = torch.randn(B, H * G, 128, device="cuda")
    c.attend(q)
    for _ in range(2):
        tok = torch.randn(B, H, 1, 128, device="cuda")
        c.decode_step(q, tok, tok)
    torch.cuda.synchronize()
    print("multi-item", mode, G, c.precision)
# 1-bit, G = 4, >= 32 chunks per CTA: the key-side lookup-table decode
# (per-unit table builds behind named barriers, several units per CTA)
cb = P.default_codebook("1b")
cfg = P.CacheConfig(d=128, bit_mode=cb.bit_mode)
B, H, T = 8, 8, 64 * 80
c = P.PagedKvCache(cfg, B, H, max_tokens=T, cb_k=cb, cb_v=cb, check_finite=False)
x = torch.randn(B, H, T, 128, device="cuda")
c.append(x, x)
q = torch.randn(B, H * 4, 128, device="cuda")
c.attend(q)
torch.cuda.synchronize()
print("1b lut", c.precision, c.n_chunks)
rng = np.random.Generator(np.random.PCG64(0))
CB.kmeans_init(rng, "2b", n_samples=4096, n_iters=2)
v = np.random.default_rng(0).standard_normal((3000, 8)).astype(np.float32)
e = np.abs(np.random.default_rng(1).standard_normal((256, 8)).astype(np.float32)) + np.float32(0.01)
kernels.match_block(v, e, kernels.entry_inv_norms(e), True)
kernels.fwht_rows(np.random.default_rng(2).standard_normal((17, 256)).astype(np.float32))
torch.cuda.synchronize()
print("sanitize run ok")
