"""Multi-process sharding on CPU (gloo, world size 2 and 4): the shard plan
covers every (batch, kv-head) unit exactly once with its whole GQA group, and
the output all-gather reassembles the single-process result bit-for-bit.

The per-shard compute here is the oracle (test infrastructure), standing in
for PagedKvCache on a GPU: the host-side plan / gather logic is what is
under test."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_18231_b200.sharding import ShardedDecoder, plan_shards


def test_plans_cover_all_units_once():
    for (B, Hkv, Hq, W) in [(16, 8, 32, 8), (16, 8, 32, 2), (1, 8, 32, 8), (2, 8, 32, 8),
                            (4, 8, 8, 4), (128, 8, 32, 8)]:
        seen = np.zeros((B, Hkv), int)
        for r in range(W):
            p = plan_shards(B, Hkv, Hq, W, r)
            seen[p.b0:p.b1, p.h0:p.h1] += 1
            assert p.local_q_heads == p.local_kv_heads * (Hq // Hkv)
        assert (seen == 1).all()
    with pytest.raises(ValueError):
        plan_shards(3, 8, 32, 2, 0)


class _OracleCache:
    """CPU stand-in for PagedKvCache (batched units, oracle compute)."""

    def __init__(self, B, Hkv, bit_mode=2):
        from oracle import oracle as orc
        from paper_2505_18231_b200.codebook import default_codebook

        cb = default_codebook(f"{bit_mode}b")
        self.units = [[orc.OracleCache(cb.entries, cb.entries, bit_mode) for _ in range(Hkv)]
                      for _ in range(B)]

    def append(self, k, v):
        for b, row in enumerate(self.units):
            for h, u in enumerate(row):
                u.append(k[b, h].numpy(), v[b, h].numpy())

    def attend(self, q):
        B = len(self.units)
        Hkv = len(self.units[0])
        G = q.shape[1] // Hkv
        out = np.zeros((B, q.shape[1], 128), np.float32)
        for b in range(B):
            for h in range(Hkv):
                out[b, h * G:(h + 1) * G] = self.units[b][h].attend(q[b, h * G:(h + 1) * G].numpy())[2]
        return torch.from_numpy(out)


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, B, Hkv, Hq, T, q, k, v, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    plan = plan_shards(B, Hkv, Hq, world, rank)
    dec = ShardedDecoder(plan, _OracleCache(plan.local_batch, plan.local_kv_heads))
    dec.append(k, v)
    out = dec.attend(q)
    if rank == 0:
        ret["out"] = out.numpy()
    dist.destroy_process_group()


@pytest.mark.parametrize("B,Hkv,Hq,world", [(2, 2, 8, 2), (1, 4, 8, 2), (4, 2, 4, 4)])
def test_sharded_decode_matches_single_process(B, Hkv, Hq, world):
    torch.manual_seed(0)
    T = 64 + 13
    k = torch.randn(B, Hkv, T, 128)
    v = torch.randn(B, Hkv, T, 128)
    q = torch.randn(B, Hq, 128)
    ref = _OracleCache(B, Hkv)
    ref.append(k, v)
    want = ref.attend(q).numpy()
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), B, Hkv, Hq, T, q, k, v, ret), nprocs=world,
             join=True)
    assert np.array_equal(ret["out"], want)


@pytest.mark.gpu
def test_nccl_gather_outputs_one_rank_with_paged_cache():
    """The NCCL all-gather path on a real GPU (one rank, so it runs on the
    one-GPU test box): ShardedDecoder over a PagedKvCache returns the local
    cache's own output, through all_gather_into_tensor into the reused
    pre-allocated buffer."""
    import paper_2505_18231_b200 as P
    from paper_2505_18231_b200.sharding import ShardedDecoder

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", world_size=1, rank=0,
                            device_id=torch.device("cuda", 0))
    try:
        B, Hkv, Hq, T = 2, 4, 16, 64 * 5 + 9
        cb = P.default_codebook("2b")
        cache = P.PagedKvCache(P.CacheConfig(d=128, bit_mode=cb.bit_mode), B, Hkv, cb_k=cb, cb_v=cb)
        dec = ShardedDecoder(plan_shards(B, Hkv, Hq, 1, 0), cache)
        g = torch.Generator(device="cuda")
        g.manual_seed(1)
        dec.append(torch.randn(B, Hkv, T, 128, device="cuda", generator=g),
                   torch.randn(B, Hkv, T, 128, device="cuda", generator=g))
        q = torch.randn(B, Hq, 128, device="cuda", generator=g)
        full = dec.attend(q)
        buf = dec._buf
        assert buf is not None and full.shape == (B, Hq, 128)
        assert torch.equal(full, cache.attend(q))
        dec.attend(q)
        assert dec._buf is buf  # reused, not re-allocated
    finally:
        dist.destroy_process_group()
