"""Debug timeline of the warp-specialized decode kernel (CTA 0) on the C2
workload: builds paper_2505_18231_b200/libnsnkv_b200_trace.so (-DNSNKV_TRACE)
beforehand (python -m paper_2505_18231_b200.build --trace) and runs with
NSNKV_LIB pointing at it.  Prints, per role, the mean cycles between the
traced events of each work item."""
import ctypes
import os
import sys
from collections import defaultdict
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
os.environ.setdefault("NSNKV_LIB", str(ROOT / "paper_2505_18231_b200" / "libnsnkv_b200_trace.so"))
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2505_18231_b200 as P  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "fast"
cfg = sys.argv[2] if len(sys.argv) > 2 else "c2"
dev = torch.device("cuda", 0)
cache = bench.build_cache(cfg, dev, seed=1, precision=prec)
B, Hq, Hkv, T, bm = bench.CONFIGS[cfg]
q = torch.randn(B, Hq, 128, device=dev)
lib = P._lib.lib
lib.nsnkv_debug_trace.restype = ctypes.c_int
lib.nsnkv_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
for _ in range(3):
    cache.attend(q)
torch.cuda.synchronize()
lib.nsnkv_debug_trace(None, 0, 1)
cache.attend(q)
torch.cuda.synchronize()
buf = np.zeros(16 * 4096, dtype=np.uint64)
lib.nsnkv_debug_trace(buf.ctypes.data, 16 * 4096, 1)
rec = buf.reshape(16, 4096)
ev_t = defaultdict(dict)
tmin = None
rows = []
for w in range(16):
    for v in rec[w]:
        v = int(v)
        if v == 0:
            break
        rows.append((w, (v >> 16) & 0xFF, v & 0xFFFF, v >> 24))
tmin = min(r[3] for r in rows)
for w, e, i, tt in rows:
    ev_t[(w, i)][e] = tt - tmin
n = len(rows)
t = np.array([r[3] for r in rows])
t0 = tmin
print(f"{n} events, span {t.max() - t0} cycles")
names = {"cons": ["start", "full", "K done", "ready", "end"],
         "prod": ["start", "free", "full", "sc/ov", "prevMMA", "Z", "issued"]}
for r in [0, 1, 4, 13, 14]:
    kind = "cons" if r < 12 else "prod"
    items = sorted(i for (rr, i) in ev_t if rr == r)
    if not items:
        continue
    if kind == "tma":
        ts = [ev_t[(r, i)][0] for i in items]
        print(f"TMA warp: {len(items)} loads, mean gap {np.mean(np.diff(ts)):.0f} cycles")
        continue
    nm = names[kind]
    d = defaultdict(list)
    starts = []
    for i in items:
        e = ev_t[(r, i)]
        if 0 in e:
            starts.append(e[0])
        for a in range(len(nm) - 1):
            if a in e and a + 1 in e:
                d[a].append(e[a + 1] - e[a])
    per = np.mean(np.diff(starts)) if len(starts) > 1 else 0
    parts = "  ".join(f"{nm[a]}->{nm[a + 1]} {np.mean(d[a]):.0f}" for a in sorted(d))
    print(f"warp {r:2d} ({kind}) items {len(items)} period {per:.0f}: {parts}")
# warp 12: MMA issue duration and TMA cadence
m_iss = [ev_t[(12, i)][1] - ev_t[(12, i)][2] for (rr, i) in ev_t if rr == 12 and 1 in ev_t[(12, i)] and 2 in ev_t[(12, i)]]
if m_iss:
    print(f"warp 12: MMA issue block mean {np.mean(m_iss):.0f} cycles (min {np.min(m_iss)}, max {np.max(m_iss)}), {len(m_iss)} items")
tl = sorted(ev_t[(12, i)][0] for (rr, i) in ev_t if rr == 12 and 0 in ev_t[(12, i)])
if len(tl) > 1:
    print(f"warp 12: TMA issue gap mean {np.mean(np.diff(tl)):.0f} cycles over {len(tl)} items")
# meta stream: issue time of item k vs producer's mfull pass (event 2 of warp 13 + k % 3)
lead = []
for (rr, i), e in ev_t.items():
    if rr == 12 and 1 in e:
        g, nloc = i % 3, i // 3
        pe = ev_t.get((13 + g, nloc), {})
        if 2 in pe:
            lead.append(pe[2] - e[1])
if lead:
    print(f"meta: producer passes mfull {np.mean(lead):.0f} cycles after the meta issue (min {np.min(lead)}, max {np.max(lead)})")
mi = sorted(ev_t[(12, i)][1] for (rr, i) in ev_t if rr == 12 and 1 in ev_t[(12, i)])
if len(mi) > 1:
    print(f"meta issue gap mean {np.mean(np.diff(mi)):.0f}; first 20 gaps {np.diff(mi)[:20].tolist()}")
d23 = [ev_t[(12, i)][3] - ev_t[(12, i)][2] for (rr, i) in ev_t if rr == 12 and 2 in ev_t[(12, i)] and 3 in ev_t[(12, i)]]
d31 = [ev_t[(12, i)][1] - ev_t[(12, i)][3] for (rr, i) in ev_t if rr == 12 and 1 in ev_t[(12, i)] and 3 in ev_t[(12, i)]]
if d23:
    print(f"meta issue: page lookup {np.mean(d23):.0f} (max {np.max(d23)}), tma issue {np.mean(d31):.0f} (max {np.max(d31)})")
# observed payload latency: warp 12 issue of item k -> consumer (warp 4 g) passes full
lat = []
for (rr, i), e in ev_t.items():
    if rr == 12 and 0 in e:
        g, nloc = i % 3, i // 3
        ce = ev_t.get((4 * g, nloc), {})
        if 1 in ce and 0 in ce:
            lat.append((ce[1] - e[0], ce[0] - e[0]))
if lat:
    a = np.array(lat)
    print(f"payload: consumer full-pass minus issue mean {a[:,0].mean():.0f} (min {a[:,0].min()}, max {a[:,0].max()}); "
          f"consumer item start minus issue mean {a[:,1].mean():.0f}")
# ready latency: producer 'issued' (item n of group g) -> consumer 'ready' of the same item
for g in range(3):
    lat = []
    for (rr, i), e in ev_t.items():
        if rr == 13 + g and 6 in e and (4 * g, i) in ev_t and 3 in ev_t[(4 * g, i)]:
            lat.append(ev_t[(4 * g, i)][3] - e[6])
    if lat:
        print(f"group {g}: consumer ready-pass minus producer issue: mean {np.mean(lat):.0f} "
              f"min {np.min(lat)} max {np.max(lat)}")
