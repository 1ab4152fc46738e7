"""GQA-aware sharding of decode attention across the GPUs of one box.

The (batch, kv-head) units of the packed cache are independent: each carries
its G = n_q_heads / n_kv_heads query heads, its pages and its residual rows
(reference: one KvCacheState per head, simulate.py:199-202; there is no
cross-head term anywhere in attention.py:83-142).  So decode shards with no
collective inside attention; the only exchange is one all-gather of the
[B_local, Hq_local, 128] outputs per step:

  * batch >= world:  contiguous batch ranges per rank (all KV heads of a
    sequence stay on one GPU -- the data-parallel serving layout);
  * batch <  world:  the KV heads of every sequence are split in contiguous
    ranges (world must divide batch * n_kv_heads into equal blocks).

Encode shards identically (each rank appends the rows of its own units).
One process per GPU, torch.distributed with NCCL for the gather (gloo works
for CPU tests).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class ShardPlan:
    world: int
    rank: int
    batch: int
    n_kv_heads: int
    n_q_heads: int
    b0: int            # batch range [b0, b1) owned by this rank
    b1: int
    h0: int            # kv-head range [h0, h1) owned by this rank
    h1: int

    @property
    def group(self) -> int:
        return self.n_q_heads // self.n_kv_heads

    @property
    def local_batch(self) -> int:
        return self.b1 - self.b0

    @property
    def local_kv_heads(self) -> int:
        return self.h1 - self.h0

    @property
    def local_q_heads(self) -> int:
        return self.local_kv_heads * self.group

    @property
    def by_batch(self) -> bool:
        return self.local_kv_heads == self.n_kv_heads

    def q_slice(self, q: torch.Tensor) -> torch.Tensor:
        """This rank's [B_local, Hq_local, d] slice of a full [B, Hq, d] query."""
        g = self.group
        return q[self.b0:self.b1, self.h0 * g:self.h1 * g]

    def kv_slice(self, x: torch.Tensor) -> torch.Tensor:
        """This rank's slice of full [B, H_kv, n, d] keys or values."""
        return x[self.b0:self.b1, self.h0:self.h1]


def plan_shards(batch: int, n_kv_heads: int, n_q_heads: int, world: int, rank: int) -> ShardPlan:
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if n_q_heads % n_kv_heads:
        raise ValueError("n_q_heads must be a multiple of n_kv_heads")
    if batch >= world:
        if batch % world:
            raise ValueError(f"batch {batch} does not split evenly over {world} ranks")
        per = batch // world
        return ShardPlan(world, rank, batch, n_kv_heads, n_q_heads,
                         rank * per, (rank + 1) * per, 0, n_kv_heads)
    # fewer sequences than GPUs: every rank takes a contiguous kv-head block
    # of one sequence
    if world % batch or n_kv_heads % (world // batch):
        raise ValueError(f"{batch} x {n_kv_heads} units do not split evenly over {world} ranks")
    per_seq = world // batch
    hb = n_kv_heads // per_seq
    b = rank // per_seq
    j = rank % per_seq
    return ShardPlan(world, rank, batch, n_kv_heads, n_q_heads, b, b + 1, j * hb, (j + 1) * hb)


def gather_buffer(plan: ShardPlan, out_local: torch.Tensor) -> torch.Tensor:
    """Pre-allocated receive buffer for gather_outputs (allocate once, reuse
    every step)."""
    return torch.empty(plan.world * out_local.numel(), dtype=out_local.dtype,
                       device=out_local.device)


def gather_outputs(plan: ShardPlan, out_local: torch.Tensor, group=None,
                   buf: torch.Tensor | None = None) -> torch.Tensor:
    """All-gather the per-rank [B_local, Hq_local, d] outputs into the full
    [B, Hq, d] tensor (one collective; equal block sizes by construction).
    `buf` (from gather_buffer) avoids an allocation per step."""
    import torch.distributed as dist

    d = out_local.shape[-1]
    if plan.world == 1 and not dist.is_initialized():
        return out_local
    flat = buf if buf is not None else gather_buffer(plan, out_local)
    if flat.numel() != plan.world * out_local.numel():
        raise ValueError("gather buffer has the wrong size")
    dist.all_gather_into_tensor(flat, out_local.contiguous().view(-1), group=group)
    blocks = flat.view(plan.world, plan.local_batch, plan.local_q_heads, d)
    if plan.by_batch:
        return blocks.reshape(plan.batch, plan.n_q_heads, d)
    per_seq = plan.world // plan.batch
    # rank r = b * per_seq + j holds heads [j * Hq_local, (j + 1) * Hq_local) of b
    return blocks.view(plan.batch, per_seq, plan.local_q_heads, d).reshape(
        plan.batch, plan.n_q_heads, d)


class ShardedDecoder:
    """One rank's share of a sharded decode: owns the local cache and turns a
    full query batch into the full output batch."""

    def __init__(self, plan: ShardPlan, local_cache, group=None):
        self.plan = plan
        self.cache = local_cache
        self.group = group
        self._buf = None

    def append(self, keys: torch.Tensor, values: torch.Tensor):
        self.cache.append(self.plan.kv_slice(keys).contiguous(),
                          self.plan.kv_slice(values).contiguous())
        return self

    def attend(self, q: torch.Tensor) -> torch.Tensor:
        out_local = self.cache.attend(self.plan.q_slice(q).contiguous())
        if self._buf is None or self._buf.numel() != self.plan.world * out_local.numel():
            self._buf = gather_buffer(self.plan, out_local)
        return gather_outputs(self.plan, out_local, self.group, self._buf)
