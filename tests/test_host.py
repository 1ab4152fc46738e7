"""Host-side logic without a GPU: codebook file format, page <-> reference
wire layout, ledger arithmetic, configuration validation, error mapping,
and the C-ABI library's exported symbols."""

from __future__ import annotations

import hashlib
import re
from pathlib import Path

import numpy as np
import pytest

from tests.conftest import ROOT, load_golden
from tests.golden.inputs import PIPELINE_CASES

CODEBOOK_SHA = {
    1: "2b099f27201e20b533061cfd2ae3a22cd09f94565f14ffb542ae8664b18e3282",
    2: "5d8f658d8c220618220abd20e0a335ec07719695dd0fae26ba1f343e099963c5",
}


@pytest.mark.parametrize("mode", [1, 2])
def test_shipped_codebooks_are_the_reference_builds(mode):
    from paper_2505_18231_b200 import codebook as cbm

    path = cbm.CODEBOOK_DIR / f"cb{mode}_seed0.nsnc"
    data = path.read_bytes()
    assert len(data) == 8209
    assert hashlib.sha256(data).hexdigest() == CODEBOOK_SHA[mode]
    cb = cbm.deserialize(data)
    assert int(cb.bit_mode) == mode and cb.seed == 0 and cb.tuned
    assert cbm.serialize(cb) == data
    if mode == 2:
        assert (cb.entries >= 0).all()


def test_codebook_format_errors():
    from paper_2505_18231_b200 import FormatError, codebook as cbm

    data = (cbm.CODEBOOK_DIR / "cb2_seed0.nsnc").read_bytes()
    with pytest.raises(FormatError):
        cbm.deserialize(b"XXXX" + data[4:])
    with pytest.raises(FormatError):
        cbm.deserialize(data[:100])
    with pytest.raises(FormatError):
        cbm.deserialize(data + b"\x00")
    bad_version = bytearray(data)
    bad_version[4] = 9
    with pytest.raises(FormatError):
        cbm.deserialize(bytes(bad_version))


def test_codebook_packed4_roundtrip():
    from paper_2505_18231_b200 import codebook as cbm

    cb = cbm.default_codebook("1b")
    e = cb.entries.astype(np.float64)
    scale = float(np.abs(e).max()) / 7.5
    levels = np.clip(np.rint(e / scale + 7.5), 0, 15).astype(np.uint8)
    packed = cbm.Codebook(entries=cb.entries, bit_mode=cb.bit_mode, seed=0, tuned=True,
                          packed4=cbm.Packed4(levels=levels, scale=np.float32(scale)))
    back = cbm.deserialize(cbm.serialize(packed))
    assert np.array_equal(back.packed4.levels, levels)
    assert np.array_equal(back.active_entries, packed.active_entries)


def test_entry_inv_norms_component_order():
    from paper_2505_18231_b200.codebook import default_codebook, entry_inv_norms
    from oracle import oracle as orc

    cb = default_codebook("2b")
    assert np.array_equal(entry_inv_norms(cb.entries), orc.entry_inv_norms(cb.entries))


@pytest.mark.parametrize("name", [c[0] for c in PIPELINE_CASES])
def test_page_wire_roundtrip_on_reference_chunks(name):
    """Every reference-serialized chunk maps into a GPU page and back to the
    identical bytes (sign-bit permutation, parameter placement, ledger)."""
    from paper_2505_18231_b200.cache import LEDGER_BYTES, PAGE_BYTES, page_to_wire, wire_to_page

    g = load_golden(f"pipeline_{name}.npz")
    for kind in ("k", "v"):
        for blob in g[f"{kind}_wire"]:
            blob = blob.tobytes()
            bm = blob[4]
            page = wire_to_page(blob, kind)
            assert page.size == PAGE_BYTES[bm]
            assert not page[LEDGER_BYTES[bm]:].any()  # padding stays zero
            assert page_to_wire(page, bm, blob[5], kind) == blob


def test_value_sign_layout_is_a_bijection():
    """Value pages order their sign bits for the ldmatrix.trans fragments:
    word 8 i + c = component c of token pair (2i, 2i+1)."""
    from paper_2505_18231_b200.cache import permute_signs_v, unpermute_signs_v

    rng = np.random.default_rng(2)
    s = rng.integers(0, 256, (3, 64, 16)).astype(np.uint8)
    w = permute_signs_v(s)
    assert w.shape == (3, 256)
    assert np.array_equal(unpermute_signs_v(w), s)
    # token 2i+1, sub j, component c lives at bit 16 + j of word 8 i + c
    t, j, c = 37, 5, 6
    assert ((w[1, 8 * (t // 2) + c] >> (16 + j)) & 1) == ((s[1, t, j] >> c) & 1)


def test_sign_permutation_is_a_bijection():
    from paper_2505_18231_b200.cache import permute_signs, unpermute_signs

    rng = np.random.default_rng(1)
    s = rng.integers(0, 256, (64, 16)).astype(np.uint8)
    w = permute_signs(s)
    assert w.shape == (64, 4)
    assert np.array_equal(unpermute_signs(w), s)
    # popcount is preserved (a permutation of the 128 bits of a token)
    pc = lambda a: np.unpackbits(a.view(np.uint8), axis=None).sum()
    assert pc(s) == pc(w.astype(np.uint32))


def test_bit_ledger_matches_reference_numbers():
    # reference README.md:123-124 and vq.py:328-356
    from paper_2505_18231_b200 import avg_bits_per_value, ledger_bytes

    assert ledger_bytes("2b") == 2292 and ledger_bytes("1b") == 1268
    assert round(avg_bits_per_value("2b"), 4) == 2.2383
    assert round(avg_bits_per_value("1b"), 4) == 1.2383


def test_cache_config_validation():
    from paper_2505_18231_b200 import BitMode, CacheConfig, ScaleStrategy, Unsupported

    cfg = CacheConfig(d=128, bit_mode="2b", strategy="s3")
    assert cfg.bit_mode is BitMode.TWO_BIT and cfg.strategy is ScaleStrategy.PARALLEL
    cfg.check_gpu_path()
    with pytest.raises(ValueError):
        CacheConfig(d=128, bit_mode="2b", residual_size=0)
    for bad in (CacheConfig(d=64, bit_mode="1b"), CacheConfig(d=128, bit_mode="1b", residual_size=32),
                CacheConfig(d=128, bit_mode="1b", dq_enabled=False),
                CacheConfig(d=128, bit_mode="1b", bypass_vq=True)):
        with pytest.raises(Unsupported):
            bad.check_gpu_path()
    assert ScaleStrategy.parse("none") is ScaleStrategy.NONE
    assert BitMode.parse("1") is BitMode.ONE_BIT


def test_status_codes_map_to_reference_exceptions():
    from paper_2505_18231_b200 import errors

    table = {-1: errors.NonPowerOfTwoDim, -2: errors.ShapeMismatch, -3: errors.IndexOutOfRange,
             -4: errors.ZeroVector, -5: errors.DegenerateProjection, -6: errors.FormatError,
             -7: errors.CudaError, -8: errors.Unsupported}
    for code, exc in table.items():
        with pytest.raises(exc):
            errors.raise_for_status(code, "x")
        assert issubclass(exc, errors.NsnKvError)
    errors.raise_for_status(0, "")


def _header_symbols() -> set[str]:
    text = (ROOT / "include" / "nsnkv_b200.h").read_text()
    return set(re.findall(r"^\s*(?:int|size_t|int64_t|const char \*|void \*)\s*(nsnkv_\w+)\(", text, re.M))


def test_c_abi_library_exports_every_header_symbol():
    import ctypes

    from paper_2505_18231_b200 import _lib

    syms = _header_symbols()
    assert len(syms) >= 14
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    for s in sorted(syms):
        assert hasattr(lib, s), s
    assert syms == set(_lib.EXPORTED)
    assert _lib.lib.nsnkv_version() == 1


def test_c_abi_rejects_bad_arguments_without_a_gpu():
    """Argument validation happens before any device work."""
    from paper_2505_18231_b200 import _lib
    from paper_2505_18231_b200.errors import NonPowerOfTwoDim, ShapeMismatch

    with pytest.raises(NonPowerOfTwoDim):
        _lib.check(_lib.lib.nsnkv_fwht_rows(None, None, 4, 12, None))
    with pytest.raises(ShapeMismatch):
        _lib.check(_lib.lib.nsnkv_match_block(None, -1, None, None, 0, None, None, None, None, None))
    assert _lib.lib.nsnkv_fwht_rows(None, None, 0, 128, None) == 0


def test_product_never_touches_the_oracle():
    pkg = ROOT / "paper_2505_18231_b200"
    for p in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")):
        text = p.read_text()
        assert "from oracle" not in text and "import oracle" not in text, p
        assert "liboracle" not in text, p


def test_oracle_builds_with_gcc():
    from oracle import oracle as orc

    lib = orc.build()
    assert Path(lib).exists()


def test_bench_step_bytes_and_clock_summary():
    """bench.py host logic without a GPU: the algorithmic bytes of the C2
    step (300.9 MB) and the clock-sample summary
    (median SM clock, throttle reasons that were active in any sample)."""
    import bench

    B, Hq, Hkv, T, bm = bench.CONFIGS["c2"]
    assert bench.step_bytes(B, Hq, Hkv, T, bm) == 300_941_312
    cs = bench.ClockSampler.__new__(bench.ClockSampler)
    cs.samples = [["1965", "1965", "Not Active", "Not Active", "Not Active", "Not Active"],
                  ["1950", "1965", "Not Active", "Not Active", "Not Active", "Active"],
                  ["1965", "1965", "Not Active", "Not Active", "Not Active", "Not Active"]]
    cs.source = "nvml"
    s = cs.summary()
    assert s["sm_mhz"] == 1965.0 and s["sm_max_mhz"] == 1965.0
    assert s["reasons"] == ["sw_power_cap"] and s["samples"] == 3


def test_precision_policy():
    """Key codewords are always hi + lo; plain-fp16 modes that are known to
    exceed the 1e-3 tolerance need an explicit opt-in."""
    from paper_2505_18231_b200.cache import PRECISIONS, check_precision, default_precision
    from paper_2505_18231_b200.errors import Unsupported

    assert default_precision(2) == "vfast" and default_precision(1) == "vfast"
    assert check_precision("precise", 1) == "precise"
    assert check_precision("vfast", 2) == "vfast"
    assert check_precision("vfast", 1) == "vfast"
    for prec, bm in (("fast", 2), ("fast", 1)):
        with pytest.raises(Unsupported):
            check_precision(prec, bm)
        assert check_precision(prec, bm, allow_inexact=True) == prec
    with pytest.raises(ValueError):
        check_precision("balanced", 2)
    assert PRECISIONS == {"precise": 0, "vfast": 1, "fast": 2}


def test_wire_field_diff_counts():
    """tests/wirediff.py classifies byte differences per field."""
    import numpy as np

    from tests.conftest import load_golden
    from tests.wirediff import compare

    g = load_golden("pipeline_2b_normal.npz")
    ref = g["k_wire"]
    got = ref.copy()
    got[0, 6 + 5] ^= 1              # one index byte
    got[1, 6 + 1024 + 3] ^= 0x81    # two sign bits
    s2 = 6 + 2048 + 36 + 80
    v = got[2, s2:s2 + 2].view("<u2")
    v[0] += 1                       # one f16 ulp
    c = compare(got, ref, 2)
    assert c["idx_flips"] == 1 and c["signs_flips"] == 2
    assert c["s2_diffs"] == 1 and c["s2_max_ulp"] == 1
