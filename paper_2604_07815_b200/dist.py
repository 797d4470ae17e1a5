"""Multi-GPU partitioning of the decode operator.

Pairs (batch element, KV head) are independent ("for each key-value
group"), so the operator shards with no collective on the data path:

* GQA: by KV head when the heads divide evenly over the ranks, else by batch;
* MLA: one shared latent head, so by batch.

Each rank holds only its shard's KV cache and index and runs the unmodified
single-GPU kernels.  ``gather_outputs`` (NCCL / gloo all_gather) assembles
head- or batch-sharded outputs for verification only; it is not part of a step.
"""
from __future__ import annotations

import torch


def shard_plan(batch: int, num_kv_heads: int, layout: str, world: int) -> dict:
    """How `world` ranks split the (batch, KV-head) pairs."""
    if world < 1:
        raise ValueError("world must be >= 1")
    if layout != "mla" and num_kv_heads % world == 0:
        return {"axis": "kv_head", "per_rank": num_kv_heads // world}
    if batch % world == 0:
        return {"axis": "batch", "per_rank": batch // world}
    raise ValueError(f"cannot shard batch={batch}, kv_heads={num_kv_heads} ({layout}) over {world} ranks evenly")


def shard_ranges(batch: int, num_kv_heads: int, layout: str, rank: int, world: int):
    """(batch slice, kv-head slice) owned by `rank`."""
    plan = shard_plan(batch, num_kv_heads, layout, world)
    k = plan["per_rank"]
    if plan["axis"] == "kv_head":
        return slice(0, batch), slice(rank * k, (rank + 1) * k)
    return slice(rank * k, (rank + 1) * k), slice(0, num_kv_heads)


def shard_workload(w, rank: int, world: int):
    """The per-rank Workload of a strong-scaled (fixed total) problem."""
    plan = shard_plan(w.batch, w.num_kv_heads, w.layout, world)
    if plan["axis"] == "kv_head":
        G = w.num_q_heads // w.num_kv_heads
        kv = plan["per_rank"]
        return w.with_(name=f"{w.name}-kvshard{rank}of{world}", num_kv_heads=kv, num_q_heads=kv * G)
    return w.with_(name=f"{w.name}-bshard{rank}of{world}", batch=plan["per_rank"])


def shard_tensor(t: torch.Tensor, bsl: slice, hsl: slice, head_dim: int | None) -> torch.Tensor:
    """Slice a [batch, heads, ...] (or [batch, ...] when head_dim is None) tensor to a shard."""
    t = t[bsl]
    if head_dim is not None:
        t = t.narrow(head_dim, hsl.start, hsl.stop - hsl.start)
    return t.contiguous()


def gather_outputs(local: torch.Tensor, axis: str, group=None) -> torch.Tensor:
    """all_gather rank shards back into the full tensor: concatenated along
    dim 1 (query / KV heads) for a KV-head shard, dim 0 for a batch shard."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    parts = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(parts, local.contiguous(), group=group)
    return torch.cat(parts, dim=1 if axis == "kv_head" else 0)
