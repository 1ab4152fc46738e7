"""Deterministic inputs of the golden fixtures (seeded PCG64, numpy's stable
Generator streams).  Shared by gen_golden.py (which runs the reference) and
the tests (which run the CUDA path and the oracle on the same inputs)."""

from __future__ import annotations

import numpy as np

D = 128


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def misaligned(g: np.random.Generator, n: int, d: int = D) -> np.ndarray:
    """Channel-scale outliers, nonzero means and 1% outlier tokens -- the
    reference's make_misaligned_tensor recipe (verify.py:616-627)."""
    scales = np.ones(d, dtype=np.float32)
    scales[:: d // 8] = 10.0
    means = np.zeros(d, dtype=np.float32)
    means[:: d // 16] = 2.0
    t = g.standard_normal((n, d), dtype=np.float32) * scales + means
    outliers = g.integers(0, n, size=max(1, n // 100))
    t[outliers] *= 50.0
    return t


def _q_roped(g: np.random.Generator, n_q: int, position: int) -> np.ndarray:
    from oracle.oracle import rope_rows, rope_table

    q = g.standard_normal((n_q, D), dtype=np.float32)
    table = rope_table(position + 1)
    return rope_rows(q, np.full(n_q, position), table)


PIPELINE_CASES = [
    # name, bit_mode, strategy, base_position, total, batches, dist, seed
    ("2b_normal", 2, 3, 0, 229, [(0, 100), (100, 229)], "normal", 11),
    ("2b_mis", 2, 3, 0, 229, [(0, 229)], "mis", 12),
    ("1b_normal", 1, 3, 0, 229, [(0, 64), (64, 65), (65, 229)], "normal", 13),
    ("1b_mis", 1, 3, 0, 229, [(0, 229)], "mis", 14),
    ("2b_base100", 2, 3, 100, 160, [(0, 160)], "normal", 15),
    ("2b_minl2", 2, 1, 0, 128, [(0, 128)], "normal", 16),
    ("1b_normmatch", 1, 2, 0, 128, [(0, 128)], "normal", 17),
    ("2b_none", 2, 0, 0, 128, [(0, 128)], "normal", 18),
    ("2b_degen", 2, 3, 0, 192, [(0, 192)], "degen", 19),
    ("1b_degen", 1, 3, 0, 192, [(0, 150), (150, 192)], "degen", 20),
]


def pipeline_inputs():
    for name, bm, strat, base, total, batches, dist, seed in PIPELINE_CASES:
        g = rng(seed)
        if dist == "normal":
            K = g.standard_normal((total, D), dtype=np.float32)
            V = g.standard_normal((total, D), dtype=np.float32)
        elif dist == "mis":
            K = misaligned(g, total)
            V = misaligned(g, total)
        else:  # degenerate chunks: identical tokens, zero rows, one-hot rows
            K = g.standard_normal((total, D), dtype=np.float32)
            V = g.standard_normal((total, D), dtype=np.float32)
            K[:64] = K[0]          # chunk 0: identical keys -> s2 clamps, zero subs
            V[:64] = V[3]
            K[64:70] = 0.0         # zero tokens -> s1 clamps
            V[70:72] = 0.0
            K[72, :] = 0.0
            K[72, 5] = 1.0         # one-hot token
            V[128:192, 8:] = 0.0   # sparse chunk -> many zero sub-vectors
        q = _q_roped(g, 4, base + total - 1)
        yield {"name": name, "bit_mode": bm, "strategy": strat, "base_position": base,
               "batches": batches, "keys": K, "values_ht": V, "q": q}


def level1_inputs():
    fwht = {}
    for d in (2, 8, 64, 128, 1024):
        fwht[d] = rng(d).standard_normal((33 if d < 1024 else 8, d), dtype=np.float32)
    match = {}
    g = rng(99)
    e = np.abs(g.standard_normal((256, 8), dtype=np.float32)) + np.float32(0.01)
    v = g.standard_normal((5000, 8), dtype=np.float32)
    match["fold"] = (v, e, True)
    g = rng(98)
    e = g.standard_normal((256, 8), dtype=np.float32) + np.float32(0.01)
    v = g.standard_normal((5000, 8), dtype=np.float32)
    match["nofold"] = (v, e, False)
    g = rng(5)
    e = g.standard_normal((256, 8), dtype=np.float32)
    e[128:] = e[:128]  # every entry duplicated: exact ties -> lowest index
    v = g.standard_normal((5000, 8), dtype=np.float32)
    match["ties"] = (v, e, False)
    g = rng(7)
    e = np.abs(g.standard_normal((256, 8), dtype=np.float32)) + np.float32(0.01)
    v = g.standard_normal((64, 8), dtype=np.float32)
    v[0] = 0.0
    v[1] = -0.0
    v[2] = 1e-13
    v[3, :4] = -1e-14
    v[4] = 1e-30
    v[5] = np.float32(3.0e30)
    match["edge"] = (v, e, True)
    return {"fwht": fwht, "match": match}


# BASELINE configs[0] (C1): 8 KV heads x (4096 + 37) tokens, GQA 4, batch 1
C1_HEADS, C1_TOKENS, C1_G = 8, 4096 + 37, 4
C1_CASES = [
    # name, bit_mode, dist, seed, distinct value codebook
    ("2b_normal", 2, "normal", 31, False),
    ("2b_mis", 2, "mis", 32, True),
    ("1b_normal", 1, "normal", 33, False),
    ("1b_mis", 1, "mis", 34, True),
]


def c1_value_entries(entries: np.ndarray, distinct: bool) -> np.ndarray:
    """Value codebook of a C1 case: the key codebook itself, or a different
    valid codebook (rows permuted by a fixed stride, scaled by 1.25) so a K/V
    codebook swap anywhere in the GPU path changes the result."""
    e = np.ascontiguousarray(entries, np.float32)
    if not distinct:
        return e
    perm = (np.arange(256) * 37 + 11) % 256
    return np.ascontiguousarray(e[perm] * np.float32(1.25))


def c1_inputs():
    for name, bm, dist, seed, distinct in C1_CASES:
        g = rng(seed)
        if dist == "normal":
            K = g.standard_normal((C1_HEADS, C1_TOKENS, D), dtype=np.float32)
            V = g.standard_normal((C1_HEADS, C1_TOKENS, D), dtype=np.float32)
        else:
            K = np.stack([misaligned(g, C1_TOKENS) for _ in range(C1_HEADS)])
            V = np.stack([misaligned(g, C1_TOKENS) for _ in range(C1_HEADS)])
        q = np.stack([_q_roped(g, C1_G, C1_TOKENS - 1) for _ in range(C1_HEADS)])
        yield {"name": name, "bit_mode": bm, "distinct_v": distinct,
               "batches": [(0, 3001), (3001, C1_TOKENS)],
               "keys": K, "values_ht": V, "q": q}


def kernels_parity_inputs():
    """The inputs of reference pkg/tests/test_kernels_parity.py:14-57, drawn
    in that file's order (make_rng = PCG64(seed); sample_standard_normal =
    rng.standard_normal((rows, cols), float32))."""
    fwht = {d: rng(d).standard_normal((33, d), dtype=np.float32) for d in (2, 8, 64, 128, 1024)}
    match = {}
    for fold in (True, False):
        g = rng(99)
        entries = np.abs(g.standard_normal((256, 8), dtype=np.float32)) + np.float32(0.01)
        if not fold:
            entries = g.standard_normal((256, 8), dtype=np.float32) + np.float32(0.01)
        vecs = g.standard_normal((50000, 8), dtype=np.float32)
        match["fold" if fold else "nofold"] = (vecs, entries, fold)
    g = rng(5)
    entries = g.standard_normal((256, 8), dtype=np.float32)
    entries[128:] = entries[:128]  # every entry duplicated
    vecs = g.standard_normal((5000, 8), dtype=np.float32)
    match["near_ties"] = (vecs, entries, False)
    return {"fwht": fwht, "match": match}
