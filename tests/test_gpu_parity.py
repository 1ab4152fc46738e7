"""GPU parity: the CUDA path (through the C ABI) against the reference's own
outputs (golden fixtures made by tests/golden/gen_golden.py) and the oracle.

Bar (SURVEY.md §8c / BASELINE.json north_star):
  * level-1 kernels: bit-exact;
  * packed chunks: reference wire bytes bit-exact (index near-tie flips are
    counted and must stay 0 on these inputs);
  * norms and means: within 1e-5 relative;
  * decode outputs: max|d out| <= 1e-3 * max|out| (fp32 accumulation).
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from tests.conftest import codebook_for, load_golden
from tests.golden.inputs import PIPELINE_CASES, level1_inputs, pipeline_inputs

pytestmark = pytest.mark.gpu

OUT_TOL = 1e-3


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# --------------------------------------------------------------------------- level 1
@pytest.mark.parametrize("d", [2, 8, 64, 128, 1024])
def test_fwht_rows_bit_exact_vs_reference(d):
    from paper_2505_18231_b200 import kernels

    g = load_golden("level1.npz")
    x = level1_inputs()["fwht"][d]
    assert sha(x) == str(g[f"fwht_in_sha_{d}"])
    assert np.array_equal(kernels.fwht_rows(x), g[f"fwht_out_{d}"])


@pytest.mark.parametrize("name", ["fold", "nofold", "ties", "edge"])
def test_match_block_bit_exact_vs_reference(name):
    from paper_2505_18231_b200 import kernels

    g = load_golden("level1.npz")
    v, e, fold = level1_inputs()["match"][name]
    inv = kernels.entry_inv_norms(e)
    assert np.array_equal(inv, g[f"match_inv_{name}"])
    idx, sg = kernels.match_block(v, e, inv, fold)
    assert np.array_equal(idx, g[f"match_idx_{name}"])
    if fold:
        assert np.array_equal(sg, g[f"match_sgn_{name}"])
    else:
        assert sg is None
    if f"cbmatch_idx_{name}" in g:
        i2, _, zm = kernels.match_rows(v, e, inv, fold)
        assert np.array_equal(i2, g[f"cbmatch_idx_{name}"])
        assert np.array_equal(zm.astype(np.uint8), g[f"cbmatch_zero_{name}"])


def test_match_block_large_vs_oracle():
    from oracle import oracle as orc
    from paper_2505_18231_b200 import kernels

    g = np.random.Generator(np.random.PCG64(2024))
    for fold in (True, False):
        e = g.standard_normal((256, 8), dtype=np.float32) + np.float32(0.01)
        if fold:
            e = np.abs(e)
        inv = orc.entry_inv_norms(e)
        v = g.standard_normal((200_000, 8), dtype=np.float32)
        a = kernels.match_block(v, e, inv, fold)
        b = orc.match_block(v, e, inv, fold)
        assert np.array_equal(a[0], b[0])
        if fold:
            assert np.array_equal(a[1], b[1])


# --------------------------------------------------------------------------- pipeline
def _run_gpu_case(case):
    from paper_2505_18231_b200 import CacheConfig, PagedKvCache, ScaleStrategy

    cb = codebook_for(case["bit_mode"])
    cfg = CacheConfig(d=128, bit_mode=cb.bit_mode, strategy=ScaleStrategy(case["strategy"]))
    cache = PagedKvCache(cfg, 1, 1, cb_k=cb, cb_v=cb, base_position=case["base_position"])
    K, V = case["keys"], case["values_ht"]
    for a, b in case["batches"]:
        cache.append(K[a:b][None, None], V[a:b][None, None])
    return cache


@pytest.mark.parametrize("case", list(pipeline_inputs()), ids=[c[0] for c in PIPELINE_CASES])
def test_encode_pages_match_reference_wire(case):
    g = load_golden(f"pipeline_{case['name']}.npz")
    assert sha(case["keys"]) == str(g["keys_sha"]) and sha(case["values_ht"]) == str(g["values_sha"])
    cache = _run_gpu_case(case)
    assert cache.n_chunks == int(g["n_chunks"]) and cache.total_tokens == int(g["total"])
    for kind in ("k", "v"):
        got = np.stack([np.frombuffer(w, np.uint8) for w in cache.chunk_wire(0, kind)])
        ref = g[f"{kind}_wire"]
        assert got.shape == ref.shape
        # index flips would show up here; there must be none on these inputs
        assert np.array_equal(got, ref), f"{kind} chunks differ at bytes {np.nonzero(got != ref)[1][:20]}"
    cnt = cache.counters()[0]
    assert list(cnt[:3]) == list(g["counters"])
    assert hashlib.sha256(cache.snapshot(0)).hexdigest() == str(g["snapshot_sha"])


@pytest.mark.parametrize("case", list(pipeline_inputs()), ids=[c[0] for c in PIPELINE_CASES])
def test_decode_matches_reference(case):
    import paper_2505_18231_b200 as P

    g = load_golden(f"pipeline_{case['name']}.npz")
    cb = codebook_for(case["bit_mode"])
    cfg = P.CacheConfig(d=128, bit_mode=cb.bit_mode, strategy=P.ScaleStrategy(case["strategy"]))
    st = P.new_cache(cfg, base_position=case["base_position"])
    for a, b in case["batches"]:
        P.append(st, case["keys"][a:b], case["values_ht"][a:b], cb, cb)
    for i, q in enumerate(case["q"]):
        s = P.scores_quantized(q, st, cb)
        ref_s = g["scores"][i]
        assert np.max(np.abs(s - ref_s)) <= 1e-5 * max(1.0, np.max(np.abs(ref_s)))
        w, out = P.attend_quantized(q, st, cb, cb)
        assert np.max(np.abs(w - g["weights"][i])) <= 1e-4 * g["weights"][i].max()
        ref_o = g["out"][i]
        assert np.max(np.abs(out - ref_o)) <= OUT_TOL * np.max(np.abs(ref_o))
        o2 = P.output_quantized(g["weights"][i], st, cb)
        assert np.max(np.abs(o2 - ref_o)) <= 1e-5 * np.max(np.abs(ref_o)) + 1e-7
    # fused batched attend (nsnkv_decode_attend)
    out_f = st.gpu.attend(case["q"][None]).cpu().numpy()[0]
    for i in range(len(case["q"])):
        ref_o = g["out"][i]
        assert np.max(np.abs(out_f[i] - ref_o)) <= OUT_TOL * np.max(np.abs(ref_o))


def test_rope_table_matches_numpy():
    import torch

    from oracle import oracle as orc
    from paper_2505_18231_b200.cache import RopeTable

    t = RopeTable(torch.device("cuda", 0), 10000.0)
    n = 140_000
    got = t.ensure(n)[:n].cpu().numpy()
    ref = orc.rope_table(n)
    mism = int((got != ref).sum())
    assert mism <= 2, f"{mism} float32 cos/sin values differ from numpy"


@pytest.mark.parametrize("case", list(pipeline_inputs()), ids=[c[0] for c in PIPELINE_CASES])
def test_fused_precision_modes_vs_reference(case):
    """Every decode precision mode usable for the case's bit mode (DESIGN.md
    §3.2) stays within the north-star output tolerance of the reference on
    every golden case, including the misaligned fixtures."""
    import torch

    import paper_2505_18231_b200 as P

    g = load_golden(f"pipeline_{case['name']}.npz")
    cb = codebook_for(case["bit_mode"])
    # key codewords are always hi + lo; value codewords may be plain fp16
    # ("vfast") in both bit modes (cache.default_precision)
    modes = ("precise", "vfast")
    for prec in modes:
        cfg = P.CacheConfig(d=128, bit_mode=cb.bit_mode, strategy=P.ScaleStrategy(case["strategy"]))
        c = P.PagedKvCache(cfg, 1, 1, cb_k=cb, cb_v=cb, base_position=case["base_position"],
                           precision=prec)
        for a, b in case["batches"]:
            c.append(torch.from_numpy(case["keys"][a:b][None, None]).cuda(),
                     torch.from_numpy(case["values_ht"][a:b][None, None]).cuda())
        out = c.attend(torch.from_numpy(case["q"][None]).cuda()).cpu().numpy()[0]
        for i in range(len(case["q"])):
            ref_o = g["out"][i]
            err = np.max(np.abs(out[i] - ref_o))
            assert err <= OUT_TOL * np.max(np.abs(ref_o)), (prec, i, err)


@pytest.mark.parametrize("mode", ["1b", "2b"])
def test_encode_exact_ties_vs_oracle(mode):
    """Codebooks with duplicated and rescaled entries make exact and
    last-bit cosine ties everywhere (reference tie rule: the lowest index
    wins, test_kernels_parity.py:41-54).  Every such sub-vector goes through
    the encode kernel's warp-cooperative fp64 pass; the pages must still be
    bit-identical to the oracle's chunks."""
    import torch

    import paper_2505_18231_b200 as P
    from oracle import oracle as orc

    base = codebook_for(int(mode[0]))
    e = base.entries.copy()
    e[1::2] = e[0::2]                                   # exact duplicates: 128 tie pairs
    e[2:64:4] = e[0:62:4] * np.float32(1.0000001)       # same direction, other norm
    cb = P.Codebook(entries=e, bit_mode=base.bit_mode)
    cfg = P.CacheConfig(d=128, bit_mode=cb.bit_mode)
    B, H, T = 1, 2, 64 * 3
    rng = np.random.default_rng(3)
    k = rng.standard_normal((B, H, T, 128)).astype(np.float32)
    v = rng.standard_normal((B, H, T, 128)).astype(np.float32)
    cache = P.PagedKvCache(cfg, B, H, cb_k=cb, cb_v=cb)
    cache.append(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    near_ties = int(cache.counters()[:, 3].sum())
    assert near_ties > 0
    for u in range(B * H):
        oc = orc.OracleCache(cb.entries, cb.entries, int(cb.bit_mode))
        oc.append(k[0, u], v[0, u])
        assert cache.chunk_wire(u, "k") == oc.k_chunks
        assert cache.chunk_wire(u, "v") == oc.v_chunks
