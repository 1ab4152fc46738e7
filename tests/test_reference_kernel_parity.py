"""The reference's own kernel bit-parity suite (pkg/tests/test_kernels_parity.py:
14-57) replayed with this package's CUDA backend in the `native` slot.

The reference suite asserts `native` == `python` bit for bit on these exact
inputs; the expected outputs here were produced by the reference itself
(tests/golden/gen_kernels_parity.py), so `cuda` == reference is the same
assertion.  The CPU half pins the oracle to the same outputs."""

from __future__ import annotations

import numpy as np
import pytest

from tests.conftest import load_golden
from tests.golden.inputs import kernels_parity_inputs

INP = kernels_parity_inputs()


def _backends():
    """The reference's kernels.backends() with the CUDA module registered."""
    from paper_2505_18231_b200 import kernels as cuda

    return {"native": cuda}


@pytest.mark.gpu
@pytest.mark.parametrize("d", [2, 8, 64, 128, 1024])
def test_fwht_bitwise_parity(d):
    g = load_golden("kernels_parity.npz")
    assert np.array_equal(_backends()["native"].fwht_rows(INP["fwht"][d]), g[f"fwht_{d}"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["fold", "nofold"])
def test_match_bitwise_parity(name):
    g = load_golden("kernels_parity.npz")
    vecs, entries, fold = INP["match"][name]
    k = _backends()["native"]
    inv = k.entry_inv_norms(entries)
    idx, sg = k.match_block(vecs, entries, inv, fold)
    assert np.array_equal(idx, g[f"match_idx_{name}"])
    if fold:
        assert np.array_equal(sg, g[f"match_sgn_{name}"])
    else:
        assert sg is None


@pytest.mark.gpu
def test_match_parity_on_near_ties():
    g = load_golden("kernels_parity.npz")
    vecs, entries, fold = INP["match"]["near_ties"]
    k = _backends()["native"]
    idx, _ = k.match_block(vecs, entries, k.entry_inv_norms(entries), fold)
    assert np.array_equal(idx, g["match_idx_near_ties"])
    assert idx.max() < 128  # ties resolve to the first copy


@pytest.mark.parametrize("name", ["fold", "nofold", "near_ties"])
def test_oracle_on_the_reference_parity_inputs(name):
    from oracle import oracle as orc

    g = load_golden("kernels_parity.npz")
    vecs, entries, fold = INP["match"][name]
    idx, sg = orc.match_block(vecs, entries, orc.entry_inv_norms(entries), fold)
    assert np.array_equal(idx, g[f"match_idx_{name}"])
    if fold:
        assert np.array_equal(sg, g[f"match_sgn_{name}"])
