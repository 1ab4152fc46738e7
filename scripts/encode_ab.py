"""C3 encode: the per-kind nsnkv_encode_chunks launches vs one nsnkv_append
launch (PagedKvCache.append), device time with CUDA events, host overhead
excluded (events recorded around the launches only)."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2505_18231_b200 as P  # noqa: E402
from paper_2505_18231_b200 import _lib  # noqa: E402

dev = torch.device("cuda", 0)
B, H, T = 64, 8, 8192
for mode in ("2b", "1b"):
    cb = P.default_codebook(mode)
    cfg = P.CacheConfig(d=128, bit_mode=cb.bit_mode)
    g = torch.Generator(device=dev)
    g.manual_seed(3)
    k = torch.randn(B, H, T, 128, device=dev, generator=g).to(torch.bfloat16)
    v = torch.randn(B, H, T, 128, device=dev, generator=g).to(torch.bfloat16)
    U, F = B * H, T // 64
    pb = P.cache.PAGE_BYTES[cb.bit_mode]
    pool = torch.empty(U * F, pb, dtype=torch.uint8, device=dev)
    ids = torch.arange(U * F, dtype=torch.int32, device=dev).view(U, F)
    res = torch.zeros(U, 64, 128, device=dev)
    start = torch.zeros(U, dtype=torch.int64, device=dev)
    table = P.cache.RopeTable.get(dev, 10000.0).ensure(T + 64)
    h = cb.device_handle(dev)
    st = torch.cuda.current_stream().cuda_stream

    def old():
        for is_key, x in ((1, k), (0, v)):
            _lib.check(_lib.lib.nsnkv_encode_chunks(res.data_ptr(), 0, x.data_ptr(), 1, T, U, F, is_key,
                                                    start.data_ptr(), table.data_ptr(), 0, table.shape[0],
                                                    h, 3, pool.data_ptr(), ids.data_ptr(), F, None, st))

    def timed(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return best

    t_old = timed(old)
    caches = [P.PagedKvCache(cfg, B, H, max_tokens=T, cb_k=cb, cb_v=cb, device=dev, check_finite=False)
              for _ in range(5)]
    host = []

    def new():
        c = caches.pop()
        t0 = time.perf_counter()
        c.append(k, v)
        host.append(time.perf_counter() - t0)
        if len(caches) == 0:  # host-side profile of one append
            import cProfile
            import pstats
            c2 = P.PagedKvCache(cfg, B, H, max_tokens=T, cb_k=cb, cb_v=cb, device=dev, check_finite=False)
            torch.cuda.synchronize()
            pr = cProfile.Profile()
            pr.enable()
            c2.append(k, v)
            pr.disable()
            pstats.Stats(pr).sort_stats("cumulative").print_stats(12)
    torch.cuda.synchronize()
    t_new = timed(new)
    print(f"{mode}: encode_chunks x2 {t_old:.3f} ms | PagedKvCache.append {t_new:.3f} ms, "
          f"host enqueue {min(host) * 1e3:.3f} ms")
    del caches
