"""The oracle (oracle/nsnkv_oracle.c) pinned against the REFERENCE's own
outputs: the golden fixtures in tests/golden were produced by running
/root/reference/pkg (see tests/golden/gen_golden.py) on the inputs that
tests/golden/inputs.py regenerates here from seeds.

Bar: level-1 kernels and packed chunks (reference wire bytes) bit-exact;
counters equal; pre-quantization norms and means within 1e-5 relative;
attention scores / weights / outputs within 1e-5 (same fp32 arithmetic,
different summation order).
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from oracle import oracle as orc
from tests.conftest import load_golden
from tests.golden.inputs import PIPELINE_CASES, level1_inputs, pipeline_inputs


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("d", [2, 8, 64, 128, 1024])
def test_oracle_fwht_bit_exact(d):
    g = load_golden("level1.npz")
    x = level1_inputs()["fwht"][d]
    assert sha(x) == str(g[f"fwht_in_sha_{d}"])
    assert np.array_equal(orc.fwht_rows(x), g[f"fwht_out_{d}"])


def test_oracle_fwht_known_answer():
    # reference test_hadamard.py:12-14: [1,1,1,1] -> [2,0,0,0] (orthonormal)
    out = orc.fwht_rows(np.ones((1, 4), np.float32))
    assert np.array_equal(out, np.array([[2, 0, 0, 0]], np.float32) * np.float32(0.5) * 2)


@pytest.mark.parametrize("name", ["fold", "nofold", "ties", "edge"])
def test_oracle_match_bit_exact(name):
    g = load_golden("level1.npz")
    v, e, fold = level1_inputs()["match"][name]
    inv = orc.entry_inv_norms(e)
    assert np.array_equal(inv, g[f"match_inv_{name}"])
    idx, sg = orc.match_block(v, e, inv, fold)
    assert np.array_equal(idx, g[f"match_idx_{name}"])
    if fold:
        assert np.array_equal(sg, g[f"match_sgn_{name}"])
    if f"cbmatch_idx_{name}" in g:
        i2, _, zm = orc.match_block(v, e, inv, fold, substitute_zero=True)
        assert np.array_equal(i2, g[f"cbmatch_idx_{name}"])
        assert np.array_equal(zm.astype(np.uint8), g[f"cbmatch_zero_{name}"])


def test_ties_resolve_to_lowest_index():
    v, e, fold = level1_inputs()["match"]["ties"]
    idx, _ = orc.match_block(v, e, orc.entry_inv_norms(e), fold)
    assert idx.max() < 128


def _oracle_case(case):
    from paper_2505_18231_b200.codebook import default_codebook

    cb = default_codebook(f"{case['bit_mode']}b")
    oc = orc.OracleCache(cb.entries, cb.entries, case["bit_mode"], strategy=case["strategy"],
                         base_position=case["base_position"])
    for a, b in case["batches"]:
        oc.append(case["keys"][a:b], case["values_ht"][a:b])
    return oc


CASES = list(pipeline_inputs())
IDS = [c[0] for c in PIPELINE_CASES]


@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_oracle_chunks_match_reference_wire(case):
    g = load_golden(f"pipeline_{case['name']}.npz")
    assert sha(case["keys"]) == str(g["keys_sha"])
    assert sha(case["values_ht"]) == str(g["values_sha"])
    assert sha(case["q"]) == str(g["q_sha"])
    oc = _oracle_case(case)
    assert len(oc.k_chunks) == int(g["n_chunks"]) and oc.total == int(g["total"])
    for kind, chunks in (("k", oc.k_chunks), ("v", oc.v_chunks)):
        got = np.stack([np.frombuffer(w, np.uint8) for w in chunks])
        assert np.array_equal(got, g[f"{kind}_wire"])
    assert list(oc.counters[:3]) == list(g["counters"])


@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_oracle_norms_and_means_within_1e5(case):
    g = load_golden(f"pipeline_{case['name']}.npz")
    oc = _oracle_case(case)
    parts = oc.nsn_k + oc.nsn_v
    for i, p in enumerate(parts):
        for key, ref in (("s1", g["nsn_s1"][i]), ("s2", g["nsn_s2"][i])):
            rel = np.abs(p[key] - ref) / np.maximum(np.abs(ref), 1e-30)
            # clamped norms are exactly NORM_EPS on both sides
            assert rel.max() <= 1e-5, key
        ref_o = g["nsn_o"][i]
        scale = max(np.abs(ref_o).max(), 1e-30)
        assert np.abs(p["o"] - ref_o).max() <= 1e-5 * scale


@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_oracle_attention_matches_reference(case):
    g = load_golden(f"pipeline_{case['name']}.npz")
    oc = _oracle_case(case)
    sc, w, out = oc.attend(case["q"])
    for i in range(len(case["q"])):
        ref_s = g["scores"][i]
        assert np.abs(sc[i] - ref_s).max() <= 1e-5 * max(1.0, np.abs(ref_s).max())
        assert np.abs(w[i] - g["weights"][i]).max() <= 1e-4 * g["weights"][i].max()
        ref_o = g["out"][i]
        assert np.abs(out[i] - ref_o).max() <= 1e-5 * np.abs(ref_o).max()


def test_f16_conversion_matches_numpy():
    rng = np.random.default_rng(0)
    vals = np.concatenate([
        rng.standard_normal(20000).astype(np.float32) * np.float32(10) ** rng.integers(-8, 6, 20000),
        np.array([0.0, -0.0, 65504, 65519.99, 65520, 1e9, -1e9, 5.96e-8, 2.98e-8, 2.9802326e-08,
                  6.1e-5, 1e-45, np.inf, -np.inf], np.float32),
    ]).astype(np.float32)
    lib = orc.lib()
    got = np.array([lib.orc_f32_to_f16(float(x)) for x in vals], np.uint16)
    assert np.array_equal(got, vals.astype(np.float16).view(np.uint16))
