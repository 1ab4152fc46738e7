"""Field-level comparison of serialized chunks (reference vq.py:363-380 wire
format) -- counts index flips, sign flips, nibble changes and f16 ulp
distances instead of a bare byte diff, so parity at BASELINE sizes can be
stated as counted, bounded differences (north_star: "any near-tie flips are
counted and bounded")."""

from __future__ import annotations

import numpy as np

R, D = 64, 128


def fields(bit_mode: int) -> dict[str, tuple[int, int, str]]:
    """name -> (offset, length, kind) of one wire chunk."""
    off = 6
    f = {"idx": (off, 1024, "u8")}
    off += 1024
    if int(bit_mode) == 2:
        f["signs"] = (off, 1024, "bits")
        off += 1024
    f["s1_par"] = (off, 4, "f16")
    off += 4
    f["s1_nib"] = (off, 32, "nib")
    off += 32
    f["o_par"] = (off, 16, "f16")
    off += 16
    f["o_nib"] = (off, 64, "nib")
    off += 64
    f["s2"] = (off, 128, "f16")
    off += 128
    f["_end"] = (off, 0, "")
    return f


def _f16_ulps(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """|ulp distance| between f16 bit patterns (sign-magnitude -> ordered)."""
    def ordered(x):
        x = x.astype(np.int32)
        return np.where(x & 0x8000, 0x8000 - (x & 0x7FFF), 0x8000 + x)
    return np.abs(ordered(a) - ordered(b))


def compare(got: np.ndarray, ref: np.ndarray, bit_mode: int) -> dict:
    """got/ref: [n_chunks, wire_bytes] u8.  Returns counters."""
    got = np.asarray(got, np.uint8).reshape(-1, ref.shape[-1])
    ref = np.asarray(ref, np.uint8).reshape(-1, ref.shape[-1])
    f = fields(bit_mode)
    assert f["_end"][0] == ref.shape[1], "wire size mismatch"
    out = {"chunks": int(ref.shape[0]), "subvectors": int(ref.shape[0]) * R * (D // 8),
           "header_diff": int((got[:, :6] != ref[:, :6]).sum())}
    for name, (o, n, kind) in f.items():
        if not n:
            continue
        g, r = got[:, o:o + n], ref[:, o:o + n]
        if kind == "u8":
            out[f"{name}_flips"] = int((g != r).sum())
        elif kind == "bits":
            out[f"{name}_flips"] = int(np.unpackbits(g ^ r).sum())
        elif kind == "nib":
            x = g ^ r
            out[f"{name}_diffs"] = int(((x & 15) != 0).sum() + ((x >> 4) != 0).sum())
        else:
            u = _f16_ulps(g.view("<u2"), r.view("<u2"))
            out[f"{name}_diffs"] = int((u != 0).sum())
            out[f"{name}_max_ulp"] = int(u.max()) if u.size else 0
    return out
