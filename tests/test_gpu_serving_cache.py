"""Serving-grade cache on the GPU: per-unit lengths,
ragged appends in one launch, page recycling, growth without copying pages,
and import of reference-serialized state.

Reference: kvcache.py:77-107 (one KvCacheState per head, own length),
kvcache.py:157-195 (append), kvcache.py:198-213 (snapshot), vq.py:363-428
(serialize / deserialize_chunk).
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest
import torch

from tests.conftest import codebook_for, load_golden
from tests.golden.inputs import pipeline_inputs

pytestmark = pytest.mark.gpu
OUT_TOL = 1e-3
CASES = {c["name"]: c for c in pipeline_inputs()}


def _cache(bm, B, H=1, **kw):
    import paper_2505_18231_b200 as P

    cb = codebook_for(bm)
    return P.PagedKvCache(P.CacheConfig(d=128, bit_mode=cb.bit_mode), B, H, cb_k=cb, cb_v=cb, **kw)


def _steps(names):
    """The golden cases' own append batches, replayed as ragged serving steps:
    step i appends batch i of every case (0 tokens once a case is done)."""
    cases = [CASES[n] for n in names]
    n_steps = max(len(c["batches"]) for c in cases)
    for i in range(n_steps):
        lens, k, v = [], [], []
        for c in cases:
            if i < len(c["batches"]):
                a, b = c["batches"][i]
                lens.append(b - a)
                k.append(c["keys"][a:b])
                v.append(c["values_ht"][a:b])
            else:
                lens.append(0)
        yield lens, np.concatenate(k)[:, None], np.concatenate(v)[:, None]


@pytest.mark.parametrize("names", [("2b_normal", "2b_mis", "2b_degen"),
                                   ("1b_normal", "1b_mis", "1b_degen")])
def test_ragged_batch_vs_reference_goldens(names):
    """Three reference streams of different lengths and batchings served as
    one ragged batch: every unit's snapshot is byte-identical to the
    reference's and the fused decode matches its attend_quantized."""
    bm = CASES[names[0]]["bit_mode"]
    c = _cache(bm, len(names))
    for lens, k, v in _steps(names):
        c.append(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), seq_lens=lens)
    for u, n in enumerate(names):
        g = load_golden(f"pipeline_{n}.npz")
        assert hashlib.sha256(c.snapshot(u)).hexdigest() == str(g["snapshot_sha"]), n
        assert c.unit_total[u] == int(g["total"])
    q = np.stack([CASES[n]["q"] for n in names])  # [3 sequences, 4 q-heads, 128]
    out = c.attend(torch.from_numpy(q).cuda()).cpu().numpy()
    for u, n in enumerate(names):
        g = load_golden(f"pipeline_{n}.npz")
        for i in range(q.shape[1]):
            ref = g["out"][i]
            assert np.max(np.abs(out[u, i] - ref)) <= OUT_TOL * np.max(np.abs(ref)), (n, i)


@pytest.mark.parametrize("name", ["2b_normal", "1b_normal", "2b_base100"])
def test_import_reference_state(name):
    """Reference-serialized chunks + residual rows imported into a unit give
    the reference's snapshot and decode (the inverse of export)."""
    case = CASES[name]
    g = load_golden(f"pipeline_{name}.npz")
    c = _cache(case["bit_mode"], 2, base_position=0)
    T = int(g["total"])
    n = int(g["n_chunks"])
    K, V = case["keys"], case["values_ht"]
    c.import_unit(1, [w.tobytes() for w in g["k_wire"]], [w.tobytes() for w in g["v_wire"]],
                  K[n * 64:T], V[n * 64:T], base_position=case["base_position"])
    assert hashlib.sha256(c.snapshot(1)).hexdigest() == str(g["snapshot_sha"])
    # snapshot -> load_snapshot round trip into the other unit
    c.load_snapshot(0, c.snapshot(1))
    assert c.snapshot(0) == c.snapshot(1)
    q = torch.from_numpy(np.stack([case["q"], case["q"]])).cuda()
    out = c.attend(q).cpu().numpy()
    for u in (0, 1):
        for i in range(case["q"].shape[0]):
            ref = g["out"][i]
            assert np.max(np.abs(out[u, i] - ref)) <= OUT_TOL * np.max(np.abs(ref))
    # appending after an import continues the reference stream
    more = torch.randn(1, 1, 70, 128, device="cuda").expand(2, 1, 70, 128).contiguous()
    c.append(more, more)
    assert c.snapshot(0) == c.snapshot(1)


def test_release_recycles_pages_and_resets_the_unit():
    B, H = 3, 2
    c = _cache(2, B, H)
    g = torch.Generator(device="cuda")
    g.manual_seed(4)
    x = torch.randn(B, H, 64 * 5 + 9, 128, device="cuda", generator=g)
    c.append(x, x)
    cap = c.capacity
    before = [c.snapshot(u) for u in range(B * H)]
    c.release([1])
    assert c.unit_total[2] == 0 and c.unit_total[3] == 0
    assert c.unit_total[0] == 64 * 5 + 9
    # a new sequence in slot 1 reuses the freed pages: no growth
    y = torch.randn(1, H, 64 * 5, 128, device="cuda", generator=g)
    packed = y[0].transpose(0, 1).contiguous()            # [rows, H, 128]
    c.append(packed, packed, seq_lens=[0, 64 * 5, 0])
    assert c.capacity == cap
    fresh = _cache(2, 1, H)
    fresh.append(y, y)
    for h in range(H):
        assert c.snapshot(2 + h) == fresh.snapshot(h)
    for u in (0, 1, 4, 5):  # other sequences untouched
        assert c.snapshot(u) == before[u]


def test_growth_never_moves_pages():
    """Pools grow by mapping memory into the reserved range: base pointers
    and existing pages stay put while the cache grows from empty."""
    c = _cache(1, 2, 2)
    g = torch.Generator(device="cuda")
    g.manual_seed(9)
    x = torch.randn(2, 2, 64 * 3, 128, device="cuda", generator=g)
    c.append(x, x)
    ptrs = c.pool_ptrs()
    first = [c.pages(u, "k").copy() for u in range(4)]
    cap0 = c.capacity
    for _ in range(4):  # 4 x 480 chunks: beyond the first mapped granules
        y = torch.randn(2, 2, 64 * 120 + 5, 128, device="cuda", generator=g)
        c.append(y, y)
    assert c.capacity > cap0
    assert c.pool_ptrs() == ptrs
    for u in range(4):
        assert np.array_equal(c.pages(u, "k")[:3], first[u])


def test_decode_step_launches_and_no_host_sync():
    """A serving decode step (1 token per sequence) adds no launch to the
    attention's two unless a chunk completes (then nsnkv_append's two);
    the loop never reads device memory (the host mirrors every length)."""
    from paper_2505_18231_b200 import _lib

    c = _cache(2, 4, 8, check_finite=False).reserve(64 * 3)
    x = torch.randn(4, 8, 64 * 2 + 60, 128, device="cuda")
    c.append(x, x)
    q = torch.randn(4, 32, 128, device="cuda")
    out = torch.empty_like(q)
    tok = torch.randn(8, 4, 8, 1, 128, device="cuda")
    torch.cuda.synchronize()
    n0 = _lib.launch_count()
    for i in range(8):  # crosses a chunk boundary (60 + 8 > 64)
        c.decode_step(q, tok[i], tok[i], out=out)
    assert _lib.launch_count() - n0 == 8 * 2 + 2  # attend + combine each step, one flush (2 launches)
    assert c.unit_n_chunks.tolist() == [3] * 32 and c.unit_n_res.tolist() == [4] * 32


@pytest.mark.parametrize("mode,G,B,H,nch", [("2b", 4, 2, 4, 2), ("1b", 8, 2, 4, 2), ("2b", 1, 2, 4, 2),
                                            ("1b", 4, 8, 8, 80)])  # the last: key-table decode
def test_decode_step_equals_append_then_attend(mode, G, B, H, nch):
    """The fused serving step (new rows attended and stored by the combine
    kernel) gives exactly the state and output of append + attend, across a
    chunk boundary (where it falls back to nsnkv_append)."""
    a = _cache(int(mode[0]), B, H, check_finite=False)
    b = _cache(int(mode[0]), B, H, check_finite=False)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(21)
    x = torch.randn(B, H, 64 * nch + 55, 128, device="cuda", generator=gen)
    a.append(x, x)
    b.append(x, x)
    for i in range(12):
        k = torch.randn(B, H, 1, 128, device="cuda", generator=gen)
        v = torch.randn(B, H, 1, 128, device="cuda", generator=gen).bfloat16()
        q = torch.randn(B, H * G, 128, device="cuda", generator=gen)
        o1 = a.decode_step(q, k, v)
        b.append(k, v)
        o2 = b.attend(q)
        assert torch.equal(o1, o2), i
    assert a.unit_n_res.tolist() == b.unit_n_res.tolist() and a.unit_n_chunks[0] == nch + 1
    for u in range(B * H):
        assert a.snapshot(u) == b.snapshot(u)
