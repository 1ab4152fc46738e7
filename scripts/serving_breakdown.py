"""Where the serving step's time goes (C2): attend alone, append alone, both;
device time per step (CUDA events) and host time per step (enqueue only)."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402

dev = torch.device("cuda", 0)
cache = bench.build_cache("c2", dev, seed=1)
B, Hq, Hkv, T, bm = bench.CONFIGS["c2"]
q = torch.randn(B, Hq, 128, device=dev)
out = torch.empty_like(q)
steps = 128
ks = torch.randn(steps, B, Hkv, 1, 128, device=dev)
vs = torch.randn(steps, B, Hkv, 1, 128, device=dev)
cache.reserve(cache.total_tokens + 4 * steps)


def run(name, fn):
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    for i in range(steps):
        fn(i)
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name:28s} device {e0.elapsed_time(e1) / steps * 1e3:8.1f} us/step   host enqueue {(t1 - t0) / steps * 1e6:8.1f} us/step")


run("attend", lambda i: cache.attend(q, out=out))
run("append (1 token)", lambda i: cache.append(ks[i], vs[i]))
run("append + attend", lambda i: (cache.append(ks[i], vs[i]), cache.attend(q, out=out)))
print("n_res", cache.n_res, "n_chunks", cache.n_chunks)
# attend cost against the residual length (exact residual rows are merged by
# the combine kernel)
for _ in range(64 - cache.n_res - 4):
    cache.append(ks[0], vs[0])
print("n_res", cache.n_res)
run("attend (residual rows)", lambda i: cache.attend(q, out=out))
