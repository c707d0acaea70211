"""KV-head sharding of the WG-KV path over N GPUs (one process per GPU).

Every object on the path is per (layer, kv head): gate MLP (gating.hpp:40-41),
HeadCache (engine.hpp:107), VS / ragged attention of the GQA group
(engine.cpp:222-240, 313-327).  Rank r of N therefore owns kv heads
[r*Hkv/N, (r+1)*Hkv/N), the q heads of their GQA groups, their gate-bank rows
and their own page pool -- no data moves between ranks except the per-layer
all-gather of head outputs that the output projection needs (SURVEY.md §5,
§8e).  The all-gather is NCCL over NVLink in production and gloo on CPU in the
tests; both go through torch.distributed.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    kv_heads: int       # local
    q_heads: int        # local
    kv_head_offset: int
    q_head_offset: int


def shard_plan(q_heads: int, kv_heads: int, world: int, rank: int) -> Shard:
    """Contiguous KV-head blocks; a GQA group never straddles ranks."""
    if kv_heads % world != 0:
        raise ValueError(f"{kv_heads} kv heads cannot be split over {world} ranks")
    if q_heads % kv_heads != 0:
        raise ValueError("q_heads must be a multiple of kv_heads (GQA, engine.cpp:224)")
    hkv = kv_heads // world
    gs = q_heads // kv_heads
    return Shard(rank, world, hkv, hkv * gs, rank * hkv, rank * hkv * gs)


def gather_heads(local_out: torch.Tensor, world: int, out: torch.Tensor | None = None) -> torch.Tensor:
    """All-gather head-sharded outputs [..., Hq/N, d] -> [..., Hq, d] (q head p at
    cols p*d as engine.cpp:234-238).  NCCL writes rank-major blocks; the final
    permute is a view-free copy only when N > 1."""
    if world == 1:
        return local_out
    lead = local_out.shape[:-2]
    shp = tuple(local_out.shape)
    flat = torch.empty((world * shp[0],) + shp[1:], dtype=local_out.dtype, device=local_out.device)
    dist.all_gather_into_tensor(flat, local_out.contiguous())  # rank-major blocks along dim 0
    buf = flat.view((world,) + shp)
    perm = list(range(1, len(lead) + 1)) + [0, len(lead) + 1, len(lead) + 2]
    full = buf.permute(*perm).reshape(*lead, world * local_out.shape[-2], local_out.shape[-1])
    if out is not None:
        out.copy_(full)
        return out
    return full
