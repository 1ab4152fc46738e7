"""BASELINE config 1 (8 KV heads x 4K tokens, GQA 4, 1-bit and 2-bit, N(0,1)
and misaligned data, distinct value codebooks on the misaligned cases) against
the REFERENCE's own outputs (tests/golden/gen_c1.py).

Packed chunks: field-level comparison with counted, bounded differences
(tests/parity_bounds.py).  Decode: max|d out| <= 1e-3 max|out| per q-head.
Fidelity (reference attention.py:53-80, test_acceptance.py:47-54 style): the
GPU output's cosine to exact attention equals the reference's within 1e-3, and
2-bit beats 1-bit (verify.py check_kvcache_monotone_fidelity).
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from tests.conftest import load_golden
from tests.golden.inputs import C1_CASES, c1_inputs, c1_value_entries
from tests.parity_bounds import check_bounds

OUT_TOL = 1e-3
CASES = list(c1_inputs())
IDS = [c[0] for c in C1_CASES]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _codebooks(case):
    import paper_2505_18231_b200 as P

    cb_k = P.default_codebook(f"{case['bit_mode']}b")
    ev = c1_value_entries(cb_k.entries, case["distinct_v"])
    cb_v = cb_k if not case["distinct_v"] else P.Codebook(entries=ev, bit_mode=cb_k.bit_mode)
    return cb_k, cb_v


def _cos(a, b):
    a = a.reshape(-1, 128).astype(np.float64)
    b = b.reshape(-1, 128).astype(np.float64)
    return (a * b).sum(1) / np.linalg.norm(a, axis=1) / np.linalg.norm(b, axis=1)


# --------------------------------------------------------------------------- CPU: oracle
@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_oracle_c1_vs_reference(case):
    """The oracle (the GPU path's bit-exact restatement) against the reference
    at C1 size: inputs regenerated exactly, differences counted and bounded,
    decode outputs within 1e-5 (same pages) of the reference's."""
    from oracle import oracle as orc

    g = load_golden(f"c1_{case['name']}.npz")
    assert sha(case["keys"]) == str(g["keys_sha"]) and sha(case["q"]) == str(g["q_sha"])
    cb_k, cb_v = _codebooks(case)
    kw, vw = [], []
    for h in range(case["keys"].shape[0]):
        oc = orc.OracleCache(cb_k.entries, cb_v.entries, case["bit_mode"])
        for a, b in case["batches"]:
            oc.append(case["keys"][h, a:b], case["values_ht"][h, a:b])
        kw.append(np.stack([np.frombuffer(c, np.uint8) for c in oc.k_chunks]))
        vw.append(np.stack([np.frombuffer(c, np.uint8) for c in oc.v_chunks]))
        assert list(oc.counters[:3]) == list(g["counters"][h])
        _, _, out = oc.attend(case["q"][h])
        for i in range(out.shape[0]):
            ref = g["out"][h, i]
            assert np.max(np.abs(out[i] - ref)) <= OUT_TOL * np.max(np.abs(ref))
    for kind, w in (("k", kw), ("v", vw)):
        c = check_bounds(np.stack(w), g[f"{kind}_wire"], case["bit_mode"])
        print(case["name"], kind, {k: v for k, v in c.items() if v})


def test_reference_fidelity_is_monotone_in_bits():
    """The goldens themselves: 2-bit decode is closer to exact attention than
    1-bit (reference check_kvcache_monotone_fidelity)."""
    c2 = _cos(load_golden("c1_2b_normal.npz")["out"], load_golden("c1_2b_normal.npz")["exact_out"])
    c1 = _cos(load_golden("c1_1b_normal.npz")["out"], load_golden("c1_1b_normal.npz")["exact_out"])
    assert c2.mean() > c1.mean() + 0.1


# --------------------------------------------------------------------------- GPU
def _gpu_cache(case, precision=None):
    import torch

    import paper_2505_18231_b200 as P

    cb_k, cb_v = _codebooks(case)
    cfg = P.CacheConfig(d=128, bit_mode=cb_k.bit_mode)
    H, T = case["keys"].shape[:2]
    c = P.PagedKvCache(cfg, 1, H, cb_k=cb_k, cb_v=cb_v, precision=precision)
    k = torch.from_numpy(case["keys"][None]).cuda()
    v = torch.from_numpy(case["values_ht"][None]).cuda()
    for a, b in case["batches"]:
        c.append(k[:, :, a:b], v[:, :, a:b])
    return c


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_gpu_c1_pages_vs_reference(case):
    g = load_golden(f"c1_{case['name']}.npz")
    c = _gpu_cache(case)
    H = case["keys"].shape[0]
    for kind in ("k", "v"):
        got = np.stack([c.wire_chunks(u, kind) for u in range(H)])
        cnt = check_bounds(got, g[f"{kind}_wire"], case["bit_mode"])
        print(case["name"], kind, {k: v for k, v in cnt.items() if v})
    assert np.array_equal(c.counters()[:, :3], g["counters"])


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_gpu_c1_decode_vs_reference_and_exact(case):
    import torch

    g = load_golden(f"c1_{case['name']}.npz")
    modes = ["precise", "vfast"]
    q = torch.from_numpy(case["q"].reshape(1, -1, 128)).cuda()
    for prec in modes:
        c = _gpu_cache(case, precision=prec)
        out = c.attend(q).cpu().numpy().reshape(g["out"].shape)
        worst = 0.0
        for h in range(out.shape[0]):
            for i in range(out.shape[1]):
                ref = g["out"][h, i]
                err = np.max(np.abs(out[h, i] - ref)) / np.max(np.abs(ref))
                worst = max(worst, err)
                assert err <= OUT_TOL, (prec, h, i, err)
        # fidelity to exact attention equals the reference's (a17)
        dc = np.abs(_cos(out, g["exact_out"]) - _cos(g["out"], g["exact_out"]))
        assert dc.max() <= 1e-3, (prec, dc.max())
        print(case["name"], prec, f"worst rel err {worst:.2e}")
