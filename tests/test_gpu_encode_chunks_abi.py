"""nsnkv_encode_chunks, the per-chunk C-ABI flush (reference
kvcache.py:114-154, flush_chunk_keys / flush_chunk_values), driven through
ctypes: every unit streams its residual rows then its fresh rows, n_flush
chunks are encoded into caller-chosen pages (scattered page ids), keys
rotated at start_pos[u] + 64 k.  Each page, converted to the reference wire
format, must equal the oracle's chunk bit for bit, and the per-chunk event
counters (clamps, zero sub-vectors, S3 fallbacks) must equal the oracle's."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode,is_key,bf16,n_resid", [("2b", 1, 0, 0), ("2b", 0, 1, 37),
                                                      ("1b", 1, 1, 63), ("1b", 0, 0, 5)])
def test_encode_chunks_vs_oracle(mode, is_key, bf16, n_resid):
    import torch

    import paper_2505_18231_b200 as P
    from paper_2505_18231_b200 import _lib
    from paper_2505_18231_b200.cache import PAGE_BYTES, RopeTable, pages_to_wire
    from oracle import oracle as orc

    rng = np.random.default_rng(11 + n_resid)
    cb = P.default_codebook(mode)
    dev = torch.device("cuda", torch.cuda.current_device())
    U, n_flush, strategy = 5, 3, 3
    n_fresh = n_flush * 64 - n_resid + 10  # 10 rows stay unflushed
    res = rng.standard_normal((U, 64, 128)).astype(np.float32)
    fresh = rng.standard_normal((U, n_fresh, 128)).astype(np.float32)
    if bf16:
        fresh = torch.from_numpy(fresh).bfloat16().float().numpy()
    start = rng.integers(0, 3000, size=U).astype(np.int64)
    table = RopeTable.get(dev, 10000.0).ensure(int(start.max()) + n_flush * 64 + 64)
    page_bytes = PAGE_BYTES[cb.bit_mode]
    n_pages = U * n_flush + 7
    pool = torch.zeros(n_pages, page_bytes, dtype=torch.uint8, device=dev)
    ids = rng.permutation(n_pages)[:U * n_flush].astype(np.int32).reshape(U, n_flush)
    res_t = torch.from_numpy(res).to(dev)
    fresh_t = torch.from_numpy(fresh).to(dev)
    if bf16:
        fresh_t = fresh_t.bfloat16()
    start_t = torch.from_numpy(start).to(dev)
    ids_t = torch.from_numpy(ids).to(dev)
    cnt_t = torch.zeros(U * n_flush, 4, dtype=torch.int32, device=dev)
    _lib.check(_lib.lib.nsnkv_encode_chunks(
        res_t.data_ptr(), n_resid, fresh_t.data_ptr(), bf16, n_fresh, U, n_flush, is_key,
        start_t.data_ptr(), table.data_ptr(), 0, table.shape[0], cb.device_handle(dev), strategy,
        pool.data_ptr(), ids_t.data_ptr(), n_flush, cnt_t.data_ptr(),
        torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    pages = pool.cpu().numpy()
    cnt = cnt_t.cpu().numpy()
    tab_np = table.cpu().numpy()  # the oracle rotates with the device table's (cos, sin)
    kind = "k" if is_key else "v"
    for u in range(U):
        stream = np.concatenate([res[u, :n_resid], fresh[u]])
        for k in range(n_flush):
            rows = stream[64 * k:64 * (k + 1)]
            p0 = int(start[u]) + 64 * k
            tab = np.ascontiguousarray(tab_np[p0:p0 + 64]) if is_key else None
            want, _, c = orc.encode_chunk(rows, bool(is_key), 0, cb.entries, int(cb.bit_mode),
                                          strategy, tab)
            got = pages_to_wire(pages[ids[u, k]], cb.bit_mode, strategy, kind)[0].tobytes()
            assert got == want, (u, k)
            # clamps, zero sub-vectors and S3 fallbacks are the reference's
            # events; the near-tie count (index 3) is the implementation's own
            # exact re-scoring, which differs between the two search designs
            assert np.array_equal(cnt[u * n_flush + k][:3], c[:3]), (u, k, cnt[u * n_flush + k], c)
