"""Multi-GPU sharding of the Quest decode path: one process per GPU.

Every reference operator reads exactly one single-head cache (kv_store.hpp:33: "paged store
... for a single attention head"), so the decode step shards over (request, KV head) units
with no exchange on the attention path.  Units are split batch-major into contiguous ranges
(a GQA group -- the query heads of one KV head -- never straddles ranks), each rank owns
the K/V pools and metadata of its units, and the only collective is the optional
all-gather of per-head outputs (NCCL over NVLink in production; any torch.distributed
backend works, the CPU tests use gloo).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class Shard:
    """Rank `rank`'s units: requests [b0, b1) x KV heads [h0, h1) (a rectangle)."""

    rank: int
    b0: int
    b1: int
    h0: int
    h1: int

    @property
    def num_requests(self) -> int:
        return self.b1 - self.b0

    @property
    def num_kv_heads(self) -> int:
        return self.h1 - self.h0

    def units(self) -> List[Tuple[int, int]]:
        return [(b, h) for b in range(self.b0, self.b1) for h in range(self.h0, self.h1)]


def partition(batch: int, num_kv_heads: int, world_size: int) -> List[Shard]:
    """Batch-major rectangular partition of the (request, KV head) units.

    world_size must divide batch * num_kv_heads in one of two ways: ranks split the batch
    (world_size divides batch: every rank serves all heads of batch/world requests) or, when
    there are fewer requests than ranks, ranks split the heads of every request (world_size
    = batch * g with g dividing num_kv_heads).  These are the layouts of SURVEY.md §8e:
    cfg3 (batch 1, 32 heads -> 32/G heads per GPU), cfg4/cfg5 (batch split first).
    """
    if batch < 1 or num_kv_heads < 1 or world_size < 1:
        raise ValueError("partition: batch, heads and world_size must be positive")
    shards = []
    if batch % world_size == 0:
        per = batch // world_size
        for r in range(world_size):
            shards.append(Shard(r, r * per, (r + 1) * per, 0, num_kv_heads))
        return shards
    if world_size % batch == 0 and num_kv_heads % (world_size // batch) == 0:
        g = world_size // batch  # ranks per request
        hp = num_kv_heads // g
        for r in range(world_size):
            b, j = divmod(r, g)
            shards.append(Shard(r, b, b + 1, j * hp, (j + 1) * hp))
        return shards
    raise ValueError(f"partition: cannot split {batch} requests x {num_kv_heads} KV heads "
                     f"evenly over {world_size} ranks")


def gather_outputs(local_out: torch.Tensor, shards: Sequence[Shard], batch: int,
                   num_kv_heads: int, group_size: int,
                   process_group: Optional[dist.ProcessGroup] = None) -> torch.Tensor:
    """All-gather every rank's [local_batch, local_kv_heads * G, d] output into the full
    [batch, num_kv_heads * G, d] tensor on every rank (G = query heads per KV head)."""
    world = dist.get_world_size(process_group)
    if world != len(shards):
        raise ValueError("gather_outputs: one shard per rank expected")
    d = local_out.shape[-1]
    # gloo has no CUDA all_gather: stage through host memory (tests, CPU-only rigs); NCCL
    # gathers device tensors directly over NVLink.
    via_host = local_out.is_cuda and dist.get_backend(process_group) == "gloo"
    src = local_out.cpu() if via_host else local_out
    parts = [torch.empty((s.num_requests, s.num_kv_heads * group_size, d), dtype=src.dtype,
                         device=src.device) for s in shards]
    # all_gather needs equal shapes: every shard of a partition has the same rectangle size.
    dist.all_gather(parts, src.contiguous(), group=process_group)
    full = torch.empty((batch, num_kv_heads * group_size, d), dtype=local_out.dtype,
                       device=local_out.device)
    for s, part in zip(shards, parts):
        full[s.b0:s.b1, s.h0 * group_size:s.h1 * group_size] = part
    return full


class ShardedDecoder:
    """One rank's slice of a model's decode path: a QuestCache holding only this rank's
    (request, KV head) units, the decode step on them, and the output gather.

    Inputs of `decode_step` are the rank's own slices (q [local_batch, local_Hq, d],
    k/v [local_batch, local_Hkv, d]); the returned tensor is the full gathered output when
    `gather=True`, else the local one.
    """

    def __init__(self, head_dim: int, page_size: int, *, num_layers: int, batch: int,
                 num_q_heads: int, num_kv_heads: int, max_tokens: int,
                 process_group: Optional[dist.ProcessGroup] = None, device: Optional[int] = None):
        from .questkv import QuestCache

        if num_q_heads % num_kv_heads:
            raise ValueError("num_q_heads must be a multiple of num_kv_heads")
        self.group = process_group
        self.rank = dist.get_rank(process_group) if dist.is_initialized() else 0
        world = dist.get_world_size(process_group) if dist.is_initialized() else 1
        self.G = num_q_heads // num_kv_heads
        self.batch, self.num_kv_heads = batch, num_kv_heads
        self.shards = partition(batch, num_kv_heads, world)
        self.shard = self.shards[self.rank]
        self.cache = QuestCache(head_dim, page_size, num_layers=num_layers,
                                max_batch=self.shard.num_requests,
                                num_q_heads=self.shard.num_kv_heads * self.G,
                                num_kv_heads=self.shard.num_kv_heads, max_tokens=max_tokens,
                                device=device)

    def local_q(self, q_full: torch.Tensor) -> torch.Tensor:
        """This rank's slice [local_batch, local_Hq, d] of a full [batch, Hq, d] query."""
        s = self.shard
        return q_full[s.b0:s.b1, s.h0 * self.G:s.h1 * self.G].contiguous()

    def local_kv(self, x_full: torch.Tensor) -> torch.Tensor:
        """This rank's slice [local_batch, local_Hkv, ...] of a full [batch, Hkv, ...] tensor."""
        s = self.shard
        return x_full[s.b0:s.b1, s.h0:s.h1].contiguous()

    def prefill(self, layer: int, seq: int, k_full: torch.Tensor, v_full: torch.Tensor,
                stream=None) -> None:
        """Bulk prefill of global sequence `seq` from all-head [Hkv, n, d] K/V (a no-op on
        ranks that do not own it)."""
        s = self.shard
        if s.b0 <= seq < s.b1:
            self.cache.prefill(layer, seq - s.b0, k_full[s.h0:s.h1].contiguous(),
                               v_full[s.h0:s.h1].contiguous(), stream=stream)

    def decode_step(self, layer: int, q: torch.Tensor, k: Optional[torch.Tensor],
                    v: Optional[torch.Tensor], token_budget: int, gather: bool = True,
                    force_include_recent: bool = True, per_layer_enabled: bool = True,
                    stream=None) -> torch.Tensor:
        out = self.cache.decode_step(layer, q, k, v, token_budget, force_include_recent,
                                     per_layer_enabled, stream=stream)
        if not gather or len(self.shards) == 1:
            return out
        return gather_outputs(out, self.shards, self.batch, self.num_kv_heads, self.G, self.group)
