"""Small end-to-end run for compute-sanitizer (memcheck / racecheck /
synccheck): encode + fused decode + unfused decode + level-1 kernels."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2505_18231_b200 as P  # noqa: E402
from paper_2505_18231_b200 import kernels  # noqa: E402

for mode, G, prec in (("2b", 4, "fast"), ("2b", 4, "precise"), ("1b", 1, None), ("2b", 8, None)):
    cb = P.default_codebook(mode)
    cfg = P.CacheConfig(d=128, bit_mode=cb.bit_mode)
    B, H, T = 2, 2, 64 * 5 + 9
    c = P.PagedKvCache(cfg, B, H, cb_k=cb, cb_v=cb, precision=prec)
    x = torch.randn(B, H, T, 128, device="cuda")
    c.append(x, x)
    q = torch.randn(B, H * G, 128, device="cuda")
    out = c.attend(q)
    s = c.scores(q)
    w = torch.softmax(s.double() / 128 ** 0.5, -1).float()
    out2 = c.output(w)
    torch.cuda.synchronize()
    print(mode, G, c.precision, float((out - out2).abs().max()))
v = np.random.default_rng(0).standard_normal((3000, 8)).astype(np.float32)
e = np.abs(np.random.default_rng(1).standard_normal((256, 8)).astype(np.float32)) + np.float32(0.01)
kernels.match_block(v, e, kernels.entry_inv_norms(e), True)
kernels.fwht_rows(np.random.default_rng(2).standard_normal((17, 256)).astype(np.float32))
torch.cuda.synchronize()
print("sanitize run ok")
