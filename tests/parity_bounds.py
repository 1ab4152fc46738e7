"""Counted-and-bounded parity against the reference at BASELINE sizes.

The encode path restates the reference operation by operation except for one
documented deviation: token norms are summed in fp64 in a fixed order where
numpy's einsum (core.py:53) uses an ISA-dependent order, so a norm can land
one f16 ulp away, and -- rarely -- a sub-vector that sits on a near-tie flips
its codeword index.  These bounds are what the tests and the
bench's ``parity`` key hold every comparison against the reference to.
"""

from __future__ import annotations

import numpy as np

from tests.wirediff import compare

# per 2^19 sub-vectors (one C1 case, 8 heads x 64 chunks x 64 tokens x 16)
MAX_IDX_FLIPS_PER_2_19 = 2
MAX_F16_ULP = 1
MAX_F16_DIFFS_PER_512_CHUNKS = 16
MAX_NIBBLE_DIFFS_PER_512_CHUNKS = 4


def check_bounds(got: np.ndarray, ref: np.ndarray, bit_mode: int) -> dict:
    """Field-level comparison of [n, W] wire chunks; asserts the bounds and
    returns the counters."""
    c = compare(got, ref, bit_mode)
    scale_sub = max(1.0, c["subvectors"] / 2 ** 19)
    scale_chunk = max(1.0, c["chunks"] / 512)
    assert c["header_diff"] == 0, c
    assert c["idx_flips"] <= MAX_IDX_FLIPS_PER_2_19 * scale_sub, c
    if "signs_flips" in c:  # a sign can only change with its sub-vector's index
        assert c["signs_flips"] <= 8 * c["idx_flips"], c
    f16 = sum(v for k, v in c.items() if k.endswith("_diffs") and not k.endswith("nib_diffs"))
    assert f16 <= MAX_F16_DIFFS_PER_512_CHUNKS * scale_chunk, c
    assert max(v for k, v in c.items() if k.endswith("_max_ulp")) <= MAX_F16_ULP, c
    nib = c["s1_nib_diffs"] + c["o_nib_diffs"]
    assert nib <= MAX_NIBBLE_DIFFS_PER_512_CHUNKS * scale_chunk, c
    return c


def summarize(counters: list[dict]) -> dict:
    """Totals over several comparisons (the bench's parity key)."""
    tot = {"subvectors": 0, "idx_flips": 0, "sign_flips": 0, "f16_diffs": 0, "f16_max_ulp": 0,
           "nibble_diffs": 0}
    for c in counters:
        tot["subvectors"] += c["subvectors"]
        tot["idx_flips"] += c["idx_flips"]
        tot["sign_flips"] += c.get("signs_flips", 0)
        tot["f16_diffs"] += sum(v for k, v in c.items()
                                if k.endswith("_diffs") and not k.endswith("nib_diffs"))
        tot["f16_max_ulp"] = max(tot["f16_max_ulp"], max(v for k, v in c.items()
                                                         if k.endswith("_max_ulp")))
        tot["nibble_diffs"] += c["s1_nib_diffs"] + c["o_nib_diffs"]
    return tot
