"""Oracle experiment behind the 1-bit "vfast" decode: decode a
1-bit cache with the value codebook rounded to fp16, with and without the
mean rounding error dbar added back, against the exact decode.  Prints the
worst max-relative output error per (context, data) case.  CPU only (oracle).
"""
import sys, numpy as np
sys.path.insert(0, '/root/repo')
from oracle import oracle as O
from tests.golden.inputs import misaligned
import glob
R, D = 64, 128
cbf = sorted(glob.glob('/root/repo/paper_2505_18231_b200/codebooks/*1*'))[0]
e, bm = O.load_nsnc_entries(cbf)
e = e.astype(np.float32)
h = e.astype(np.float16).astype(np.float32)
dbar = (e - h).mean(axis=0)   # mean rounding error per component
def run(T, mis, seed):
    g = np.random.default_rng(seed)
    K = misaligned(g, T) if mis else g.standard_normal((T, D)).astype(np.float32)
    V = misaligned(g, T) if mis else g.standard_normal((T, D)).astype(np.float32)
    V = O.fwht_rows(V)
    n = T // R
    kw = O.encode_many_pos(K.reshape(n, R, D), True, np.arange(n) * R, e, bm)
    vw = O.encode_many(V.reshape(n, R, D), False, e, bm)
    q = g.standard_normal((1, 4, D)).astype(np.float32)
    ref = O.attend_many(kw, vw, 1, n, e, e, bm, q)[0]
    res = {}
    for name, ev in (("fp16", h), ("fp16+dbar", h + dbar[None, :])):
        out = O.attend_many(kw, vw, 1, n, e, ev.astype(np.float32), bm, q)[0]
        res[name] = max(np.abs(out[i] - ref[i]).max() / np.abs(ref[i]).max() for i in range(4))
    return res
for T in (4096, 32768):
    for mis in (False, True):
        r = [run(T, mis, s) for s in range(3)]
        print(T, "mis" if mis else "n01", {k: f"{max(x[k] for x in r):.2e}" for k in r[0]})
