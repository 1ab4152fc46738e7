"""The two reusable 256x8 codebooks: file format, validation and device upload.

Runtime half of reference pkg/src/nsnkv/codebook.py:
  * ``BitMode``                 codebook.py:32-45
  * ``Packed4``                 codebook.py:57-68 (optional 4-bit entries)
  * ``Codebook``                codebook.py:71-106 (validation, active_entries,
                                inv_norms)
  * ``deserialize`` / ``load``  codebook.py:384-432 (NSNC little-endian format)
  * ``serialize`` / ``save``    codebook.py:370-381, 425-427
Building codebooks (K-Means + tuning, codebook.py:175-340) is offline and out
of scope; the seed-0 tuned codebooks the reference CLI produces ship in
``codebooks/`` (sha256 recorded in DESIGN.md).
"""

from __future__ import annotations

import ctypes
import enum
import struct
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .errors import FormatError, ShapeMismatch

N_ENTRIES = 256
ENTRY_DIM = 8
MAGIC = b"NSNC"
VERSION = 1
_HEADER = struct.Struct("<HBQB")  # version, bit mode, seed, tuned

CODEBOOK_DIR = Path(__file__).resolve().parent / "codebooks"


class BitMode(enum.IntEnum):
    ONE_BIT = 1
    TWO_BIT = 2

    @property
    def folded(self) -> bool:
        """Two-bit mode stores signs separately and matches |v|."""
        return self is BitMode.TWO_BIT

    @staticmethod
    def parse(s) -> "BitMode":
        if isinstance(s, BitMode):
            return s
        key = str(s).lower()
        table = {"1b": BitMode.ONE_BIT, "1": BitMode.ONE_BIT,
                 "2b": BitMode.TWO_BIT, "2": BitMode.TWO_BIT}
        if key not in table:
            raise ValueError(f"unknown bit mode {s!r}")
        return table[key]


def entry_inv_norms(entries: np.ndarray) -> np.ndarray:
    """fp64 1/||e|| with the squares accumulated in component order
    (reference kernels/__init__.py:44-51): the match scores depend on it."""
    e = np.asarray(entries, dtype=np.float64)
    acc = e[:, 0] * e[:, 0]
    for k in range(1, e.shape[1]):
        acc = acc + e[:, k] * e[:, k]
    return 1.0 / np.sqrt(acc)


@dataclass
class Packed4:
    """4-bit entry levels under one scale (codebook.py:57-68)."""

    levels: np.ndarray  # (256, 8) uint8
    scale: float

    def dequantized(self, bit_mode: BitMode) -> np.ndarray:
        lv = self.levels.astype(np.float32)
        if bit_mode is BitMode.TWO_BIT:
            return lv * np.float32(self.scale)
        return (lv - np.float32(7.5)) * np.float32(self.scale)


@dataclass
class Codebook:
    entries: np.ndarray
    bit_mode: BitMode
    seed: int = 0
    tuned: bool = False
    packed4: Packed4 | None = None
    _handles: dict = field(default_factory=dict, repr=False, compare=False)

    def __post_init__(self):
        e = np.ascontiguousarray(self.entries, dtype=np.float32)
        if e.shape != (N_ENTRIES, ENTRY_DIM):
            raise ValueError(f"codebook must be {N_ENTRIES}x{ENTRY_DIM}, got {e.shape}")
        self.bit_mode = BitMode.parse(self.bit_mode)
        if self.bit_mode is BitMode.TWO_BIT and (e < 0).any():
            raise ValueError("two-bit codebook entries must be nonnegative")
        if (np.sqrt((e.astype(np.float64) ** 2).sum(axis=1)) < 1e-12).any():
            raise ValueError("codebook contains a zero entry")
        self.entries = e

    @property
    def active_entries(self) -> np.ndarray:
        """Entries used by match and lookup: the 4-bit form when present."""
        if self.packed4 is None:
            return self.entries
        return self.packed4.dequantized(self.bit_mode)

    @property
    def inv_norms(self) -> np.ndarray:
        return entry_inv_norms(self.active_entries)

    # -- device upload ----------------------------------------------------
    def device_handle(self, device=None) -> int:
        """Opaque nsnkv_codebook* on ``device`` (uploaded once, cached)."""
        import torch

        from ._lib import c_void_p, check, lib

        from .cache import resolve_device

        dev = resolve_device(device)
        key = dev.index
        h = self._handles.get(key)
        if h is None:
            ent = np.ascontiguousarray(self.active_entries, dtype=np.float32)
            inv = np.ascontiguousarray(self.inv_norms, dtype=np.float64)
            out = c_void_p()
            with torch.cuda.device(dev):
                check(lib.nsnkv_codebook_create(ent.ctypes.data, inv.ctypes.data,
                                                int(self.bit_mode), ctypes.byref(out)))
            h = self._handles[key] = out.value
        return h

    def __del__(self):  # pragma: no cover - interpreter shutdown order varies
        try:
            from ._lib import lib

            for h in self._handles.values():
                lib.nsnkv_codebook_destroy(h)
            self._handles.clear()
        except Exception:
            pass


def _pack_nibbles(levels: np.ndarray) -> np.ndarray:
    v = np.asarray(levels, dtype=np.uint8).ravel()
    if v.size % 2:
        v = np.concatenate([v, np.zeros(1, np.uint8)])
    return (v[0::2] | (v[1::2] << 4)).astype(np.uint8)


def _unpack_nibbles(packed: np.ndarray, n: int) -> np.ndarray:
    p = np.asarray(packed, dtype=np.uint8)
    out = np.empty(p.size * 2, np.uint8)
    out[0::2] = p & 0x0F
    out[1::2] = p >> 4
    return out[:n]


def serialize(cb: Codebook) -> bytes:
    parts = [MAGIC, _HEADER.pack(VERSION, int(cb.bit_mode), int(cb.seed), int(cb.tuned)),
             cb.entries.astype("<f4", copy=False).tobytes()]
    if cb.packed4 is None:
        parts.append(b"\x00")
    else:
        parts += [b"\x01", struct.pack("<f", float(cb.packed4.scale)),
                  _pack_nibbles(cb.packed4.levels).tobytes()]
    return b"".join(parts)


def deserialize(data: bytes) -> Codebook:
    if len(data) < 4 or data[:4] != MAGIC:
        raise FormatError("bad codebook file: missing magic")
    pos = 4
    try:
        version, mode_raw, seed, tuned = _HEADER.unpack_from(data, pos)
    except struct.error as e:
        raise FormatError(f"bad codebook file: truncated header ({e})") from e
    pos += _HEADER.size
    if version != VERSION:
        raise FormatError(f"unsupported codebook version {version}")
    try:
        mode = BitMode(mode_raw)
    except ValueError as e:
        raise FormatError(f"bad bit mode {mode_raw}") from e
    nbytes = N_ENTRIES * ENTRY_DIM * 4
    if len(data) < pos + nbytes + 1:
        raise FormatError("bad codebook file: truncated entries")
    entries = np.frombuffer(data, "<f4", N_ENTRIES * ENTRY_DIM, pos).reshape(N_ENTRIES, ENTRY_DIM)
    pos += nbytes
    flag = data[pos]
    pos += 1
    if flag not in (0, 1):
        raise FormatError(f"bad packed4 flag {flag}")
    packed = None
    if flag:
        nn = N_ENTRIES * ENTRY_DIM // 2
        if len(data) < pos + 4 + nn:
            raise FormatError("bad codebook file: truncated packed block")
        (scale,) = struct.unpack_from("<f", data, pos)
        pos += 4
        lv = _unpack_nibbles(np.frombuffer(data, np.uint8, nn, pos), N_ENTRIES * ENTRY_DIM)
        pos += nn
        packed = Packed4(levels=lv.reshape(N_ENTRIES, ENTRY_DIM), scale=np.float32(scale))
    if pos != len(data):
        raise FormatError("bad codebook file: trailing bytes")
    return Codebook(entries=entries.astype(np.float32), bit_mode=mode, seed=int(seed),
                    tuned=bool(tuned), packed4=packed)


def load_codebook(path) -> Codebook:
    return deserialize(Path(path).read_bytes())


def save_codebook(path, cb: Codebook) -> None:
    Path(path).write_bytes(serialize(cb))


def default_codebook(bit_mode) -> Codebook:
    """The shipped seed-0 tuned codebook for a bit mode (reference CLI
    ``nsnkv build-codebook --bit-mode {1b,2b} --seed 0``)."""
    mode = BitMode.parse(bit_mode)
    return load_codebook(CODEBOOK_DIR / f"cb{int(mode)}_seed0.nsnc")


def check_entries_shape(entries: np.ndarray) -> None:
    if entries.shape != (N_ENTRIES, ENTRY_DIM):
        raise ShapeMismatch(f"expected ({N_ENTRIES}, {ENTRY_DIM}) entries, got {entries.shape}")
