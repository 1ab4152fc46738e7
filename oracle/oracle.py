"""ctypes/numpy front end of the C oracle (nsnkv_oracle.c).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Restates the reference
(/root/reference/pkg, package nsnkv):
  rope_table        rope.py:29-51 (numpy, the reference's own formula)
  fwht_rows         kernels/_native.pyx:16-38
  match_block       kernels/_native.pyx:41-87 (+ codebook.py:109-128)
  encode_chunk      kvcache.py:114-154 -> vq.serialize_chunk wire bytes
  OracleCache       kvcache.py:157-195 residual policy + attention.py:83-142
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "liboracle.so"
D, R, NPAIR = 128, 64, 64


def build(force: bool = False) -> Path:
    src = HERE / "nsnkv_oracle.c"
    if force or not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE), "_build/liboracle.so"], check=True)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(LIB))
        P = ctypes.c_void_p
        i32, i64 = ctypes.c_int32, ctypes.c_int64
        L.orc_fwht_rows.argtypes = [P, P, i64, i32]
        L.orc_match_block.argtypes = [P, i64, P, P, i32, P, P, P]
        L.orc_entry_inv_norms.argtypes = [P, P]
        L.orc_wire_bytes.argtypes = [i32]
        L.orc_wire_bytes.restype = i32
        L.orc_encode_chunk.argtypes = [P, i32, P, P, P, i32, i32, P, P, P]
        L.orc_attend.argtypes = [P, P, i32, P, P, i32, i64, P, P, P, i32, P, i32, P, P, P]
        L.orc_encode_many.argtypes = [P, i64, i32, P, P, P, i32, i32, P, i32]
        L.orc_attend_many.argtypes = [P, P, i64, i32, P, P, P, i32, P, i32, P, i32]
        L.orc_encode_many_pos.argtypes = [P, i64, i32, P, P, P, P, i32, i32, P, i32]
        L.orc_f32_to_f16.argtypes = [ctypes.c_float]
        L.orc_f32_to_f16.restype = ctypes.c_uint16
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data if a is not None else None


def wire_bytes(bit_mode: int) -> int:
    return 6 + 1024 + (1024 if int(bit_mode) == 2 else 0) + 36 + 80 + 128


# -- rope.py:29-51 -----------------------------------------------------------
def pair_freqs(d: int = D, base: float = 10000.0) -> np.ndarray:
    j = np.arange(d // 2, dtype=np.float64)
    return float(base) ** (-2.0 * j / d)


def rope_table(n_pos: int, base: float = 10000.0, pos0: int = 0) -> np.ndarray:
    """[n_pos, 64, 2] float32 (cos, sin) of float64 angles, as rope_rows does."""
    pos = np.arange(pos0, pos0 + n_pos, dtype=np.float64)
    theta = pos[:, None] * pair_freqs(D, base)[None, :]
    out = np.empty((n_pos, NPAIR, 2), np.float32)
    out[:, :, 0] = np.cos(theta).astype(np.float32)
    out[:, :, 1] = np.sin(theta).astype(np.float32)
    return out


def rope_rows(t: np.ndarray, positions, table: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(t, np.float32)
    cs = table[np.asarray(positions, dtype=np.int64)]
    c, s = cs[:, :, 0], cs[:, :, 1]
    out = np.empty_like(a)
    e, o = a[:, 0::2], a[:, 1::2]
    out[:, 0::2] = e * c - o * s
    out[:, 1::2] = e * s + o * c
    return out


# -- level 1 -------------------------------------------------------------------
def fwht_rows(a: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(a, np.float32)
    out = np.empty_like(x)
    lib().orc_fwht_rows(_p(x), _p(out), x.shape[0], x.shape[1])
    return out


def entry_inv_norms(entries: np.ndarray) -> np.ndarray:
    e = np.ascontiguousarray(entries, np.float32)
    inv = np.empty(256, np.float64)
    lib().orc_entry_inv_norms(_p(e), _p(inv))
    return inv


def match_block(vecs, entries, inv, fold: bool, substitute_zero: bool = False):
    v = np.ascontiguousarray(vecs, np.float32)
    e = np.ascontiguousarray(entries, np.float32)
    iv = np.ascontiguousarray(inv, np.float64)
    m = v.shape[0]
    idx = np.empty(m, np.uint8)
    sg = np.empty(m, np.uint8) if fold else None
    zm = np.empty(m, np.uint8) if substitute_zero else None
    lib().orc_match_block(_p(v), m, _p(e), _p(iv), int(bool(fold)), _p(idx), _p(sg), _p(zm))
    if substitute_zero:
        return idx, sg, zm.astype(bool)
    return idx, sg


# -- encode ----------------------------------------------------------------------
def encode_chunk(rows: np.ndarray, is_key: bool, start_pos: int, entries: np.ndarray,
                 bit_mode: int, strategy: int = 3, table: np.ndarray | None = None):
    """One flushed chunk -> (wire bytes, dict of s1/o/s2/s2adj, counters[4])."""
    x = np.ascontiguousarray(rows, np.float32).reshape(R, D)
    e = np.ascontiguousarray(entries, np.float32)
    inv = entry_inv_norms(e)
    cs = None
    if is_key:
        if table is None:
            cs = rope_table(R, pos0=start_pos)
        else:
            cs = np.ascontiguousarray(table[start_pos:start_pos + R])
    wire = np.empty(wire_bytes(bit_mode), np.uint8)
    nsn = np.empty(R + D + R + R, np.float32)
    cnt = np.empty(4, np.int32)
    lib().orc_encode_chunk(_p(x), int(bool(is_key)), _p(cs), _p(e), _p(inv), int(bit_mode),
                           int(strategy), _p(wire), _p(nsn), _p(cnt))
    parts = {"s1": nsn[:R].copy(), "o": nsn[R:R + D].copy(), "s2": nsn[R + D:2 * R + D].copy(),
             "s2adj": nsn[2 * R + D:].copy()}
    return wire.tobytes(), parts, cnt


class OracleCache:
    """One reference KvCacheState restated: residual policy of
    kvcache.py:157-195 with chunks kept as reference wire bytes."""

    def __init__(self, cb_k_entries, cb_v_entries, bit_mode: int, strategy: int = 3,
                 base_position: int = 0, rope_base: float = 10000.0):
        self.ek = np.ascontiguousarray(cb_k_entries, np.float32)
        self.ev = np.ascontiguousarray(cb_v_entries, np.float32)
        self.bit_mode = int(bit_mode)
        self.strategy = int(strategy)
        self.base = int(base_position)
        self.rope_base = rope_base
        self.k_chunks: list[bytes] = []
        self.v_chunks: list[bytes] = []
        self.k_res = np.zeros((0, D), np.float32)
        self.v_res = np.zeros((0, D), np.float32)
        self.total = 0
        self.counters = np.zeros(4, np.int64)
        self.nsn_k: list[dict] = []
        self.nsn_v: list[dict] = []

    def append(self, keys, values):
        k = np.ascontiguousarray(keys, np.float32)
        v = np.ascontiguousarray(values, np.float32)
        self.k_res = np.concatenate([self.k_res, k])
        self.v_res = np.concatenate([self.v_res, v])
        self.total += k.shape[0]
        while self.k_res.shape[0] >= R:
            start = self.base + len(self.k_chunks) * R
            table = rope_table(R, self.rope_base, pos0=start)
            wk, pk, ck = encode_chunk(self.k_res[:R], True, 0, self.ek, self.bit_mode,
                                      self.strategy, table)
            wv, pv, cv = encode_chunk(self.v_res[:R], False, 0, self.ev, self.bit_mode,
                                      self.strategy)
            self.k_chunks.append(wk)
            self.v_chunks.append(wv)
            self.nsn_k.append(pk)
            self.nsn_v.append(pv)
            self.counters += ck + cv
            self.k_res = self.k_res[R:]
            self.v_res = self.v_res[R:]
        return self

    def attend(self, q: np.ndarray):
        """q [G, 128] RoPE'd -> (scores [G,T], weights [G,T], out [G,128])."""
        qq = np.ascontiguousarray(q, np.float32).reshape(-1, D)
        G = qq.shape[0]
        T = self.total
        table = rope_table(self.base + T + 1, self.rope_base)
        kw = np.frombuffer(b"".join(self.k_chunks), np.uint8) if self.k_chunks else np.zeros(1, np.uint8)
        vw = np.frombuffer(b"".join(self.v_chunks), np.uint8) if self.v_chunks else np.zeros(1, np.uint8)
        kr = np.ascontiguousarray(self.k_res) if self.k_res.shape[0] else np.zeros((1, D), np.float32)
        vr = np.ascontiguousarray(self.v_res) if self.v_res.shape[0] else np.zeros((1, D), np.float32)
        sc = np.empty((G, max(T, 1)), np.float32)
        w = np.empty((G, max(T, 1)), np.float32)
        out = np.empty((G, D), np.float32)
        lib().orc_attend(_p(kw), _p(vw), len(self.k_chunks), _p(kr), _p(vr),
                         self.k_res.shape[0], self.base, _p(table), _p(self.ek), _p(self.ev),
                         self.bit_mode, _p(qq), G, _p(sc), _p(w), _p(out))
        return sc[:, :T], w[:, :T], out


def encode_many(rows: np.ndarray, is_key: bool, entries, bit_mode: int, strategy: int = 3,
                threads: int | None = None) -> np.ndarray:
    """CPU baseline: n independent chunks [n, 64, 128], keys at position 0."""
    x = np.ascontiguousarray(rows, np.float32)
    n = x.shape[0]
    e = np.ascontiguousarray(entries, np.float32)
    inv = entry_inv_norms(e)
    cs = rope_table(R) if is_key else None
    wire = np.empty((n, wire_bytes(bit_mode)), np.uint8)
    lib().orc_encode_many(_p(x), n, int(bool(is_key)), _p(cs), _p(e), _p(inv), int(bit_mode),
                          int(strategy), _p(wire), threads or os.cpu_count() or 1)
    return wire


def encode_many_pos(rows: np.ndarray, is_key: bool, pos0: np.ndarray, entries, bit_mode: int,
                    strategy: int = 3, rope_base: float = 10000.0,
                    threads: int | None = None) -> np.ndarray:
    """n chunks [n, 64, 128]; chunk i starts at absolute position pos0[i]
    (keys are rotated there, kvcache.py:114-136) -> wire chunks [n, W]."""
    x = np.ascontiguousarray(rows, np.float32)
    n = x.shape[0]
    e = np.ascontiguousarray(entries, np.float32)
    inv = entry_inv_norms(e)
    p0 = np.ascontiguousarray(pos0, np.int64)
    cs = rope_table(int(p0.max()) + R, rope_base) if is_key and n else None
    wire = np.empty((n, wire_bytes(bit_mode)), np.uint8)
    lib().orc_encode_many_pos(_p(x), n, int(bool(is_key)), _p(cs), _p(p0), _p(e), _p(inv),
                              int(bit_mode), int(strategy), _p(wire), threads or os.cpu_count() or 1)
    return wire


def attend_many(kw: np.ndarray, vw: np.ndarray, n_units: int, n_chunks: int, ent_k, ent_v,
                bit_mode: int, q: np.ndarray, threads: int | None = None) -> np.ndarray:
    """CPU baseline: n_units units of n_chunks wire chunks, G queries each."""
    G = q.shape[1]
    table = rope_table(n_chunks * R + 1)
    out = np.empty((n_units, G, D), np.float32)
    qq = np.ascontiguousarray(q, np.float32)
    lib().orc_attend_many(_p(kw), _p(vw), n_units, n_chunks, _p(table),
                          _p(np.ascontiguousarray(ent_k, np.float32)),
                          _p(np.ascontiguousarray(ent_v, np.float32)), int(bit_mode), _p(qq), G,
                          _p(out), threads or os.cpu_count() or 1)
    return out


# -- codebook.py:384-432 (NSNC file) ------------------------------------------
def load_nsnc_entries(path) -> tuple[np.ndarray, int]:
    """(active entries [256, 8] float32, bit mode) of an NSNC codebook file,
    read without the product package (the bench's reference arm must not load
    it).  Layout: b"NSNC", <u16 version, u8 bit mode, u64 seed, u8 tuned>,
    256x8 <f4 entries, u8 packed4 flag [, <f4 scale, 1024 nibble bytes]>.
    With a packed4 block the active entries are its dequantized levels
    (codebook.py:57-68)."""
    import struct

    data = Path(path).read_bytes()
    if data[:4] != b"NSNC":
        raise ValueError("not an NSNC codebook")
    version, mode, _seed, _tuned = struct.unpack_from("<HBQB", data, 4)
    pos = 4 + 12
    e = np.frombuffer(data, "<f4", 2048, pos).reshape(256, 8).astype(np.float32)
    pos += 8192
    if data[pos]:
        (scale,) = struct.unpack_from("<f", data, pos + 1)
        b = np.frombuffer(data, np.uint8, 1024, pos + 5)
        lv = np.empty(2048, np.float32)
        lv[0::2] = b & 15
        lv[1::2] = b >> 4
        lv = lv.reshape(256, 8)
        e = lv * np.float32(scale) if mode == 2 else (lv - np.float32(7.5)) * np.float32(scale)
    return np.ascontiguousarray(e, np.float32), int(mode)
