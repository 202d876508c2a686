"""Row-sharded multi-GPU search.

Database rows shard naturally: every (query, vector) distance is independent,
so rank r scans its contiguous shard [r0, r1) (whole layout-v1 groups, r0 % 8
== 0) and produces u64 keys with global indices (index_base = r0).  The only
exchange is one all-gather of the [Q][k] key lists over NCCL (NVLink /
NVSwitch), followed by the exact merge (bolt_topk_merge): keys are a total
order, so the merged result equals the single-GPU result bit for bit.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row range of `rank`: starts on a multiple of 8 (a layout-v1
    group boundary), ranges cover [0, n_total) without overlap."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    per = -(-n_total // world)
    per = -(-per // 8) * 8
    r0 = min(rank * per, n_total)
    r1 = min(r0 + per, n_total)
    return r0, r1


def gather_keys(keys: torch.Tensor, group=None) -> torch.Tensor:
    """[nq][k] u64 keys of every rank -> [W][nq][k] (all_gather_into_tensor).
    The collective moves the bits as int64 (backends lack unsigned 64-bit)."""
    world = dist.get_world_size(group)
    src = keys.contiguous().view(torch.int64)
    out = torch.empty((world * keys.shape[0],) + tuple(keys.shape[1:]), dtype=torch.int64, device=keys.device)
    dist.all_gather_into_tensor(out, src, group=group)
    return out.view(torch.uint64).view((world,) + tuple(keys.shape))


def sharded_topk(codes_shard: torch.Tensor, n_shard: int, qluts: torch.Tensor, k: int, metric,
                 index_base: int, group=None, variant: int = 0) -> torch.Tensor:
    """Top-k over the union of all ranks' shards (every rank gets the result)."""
    from . import topk, topk_merge
    local = topk(codes_shard, n_shard, qluts, k, metric, index_base=index_base, variant=variant)
    if dist.get_world_size(group) == 1:
        return local
    return topk_merge(gather_keys(local, group))
