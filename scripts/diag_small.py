import time, torch, numpy as np, sys
sys.path.insert(0, '.')
import paper_2505_18231_b200 as P
cb = P.default_codebook('2b')
cfg = P.CacheConfig(d=128, bit_mode=cb.bit_mode)
for (B, Hkv, G, T) in [(1,1,1,128), (2,2,4,213), (1,1,1,64), (4,8,4,4096)]:
    cache = P.PagedKvCache(cfg, B, Hkv, max_tokens=T, cb_k=cb, cb_v=cb)
    cache.append(torch.randn(B, Hkv, T, 128, device='cuda'), torch.randn(B, Hkv, T, 128, device='cuda'))
    torch.cuda.synchronize()
    q = torch.randn(B, Hkv * G, 128, device='cuda')
    for rep in range(3):
        t0 = time.perf_counter(); out = cache.attend(q); torch.cuda.synchronize(); dt = time.perf_counter() - t0
        print(B, Hkv, G, T, 'attend %.3f ms' % (dt * 1e3), flush=True)
