"""Multi-GPU search: row-sharded and query-sharded (8(f4)).

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


def _all_gather_into(out: torch.Tensor, src: torch.Tensor, group=None) -> None:
    """all_gather_into_tensor; under gloo (CPU collectives: the multi-process
    glue tests, and bench.py --dist-backend gloo with several ranks on one
    GPU) device tensors travel through host copies."""
    if dist.get_backend(group) == "gloo" and src.is_cuda:
        host = torch.empty(out.shape, dtype=out.dtype)
        dist.all_gather_into_tensor(host, src.cpu(), group=group)
        out.copy_(host)
    else:
        dist.all_gather_into_tensor(out, src, group=group)


def gather_keys(keys: torch.Tensor, group=None) -> torch.Tensor:
    """[nq][k] u64 keys of every rank -> [W][nq][k] (all_gather_into_tensor).
    The collective moves the bits as int64 (backends lack unsigned 64-bit)."""
    world = dist.get_world_size(group)
    src = keys.contiguous().view(torch.int64)
    out = torch.empty((world * keys.shape[0],) + tuple(keys.shape[1:]), dtype=torch.int64, device=keys.device)
    _all_gather_into(out, src, group)
    return out.view(torch.uint64).view((world,) + tuple(keys.shape))


def gather_codes(codes: torch.Tensor, n_local: int, m: int, group=None) -> tuple[torch.Tensor, int]:
    """Every rank's layout-v1 code words -> the whole database's words on every
    rank, in rank (= row) order, and the total row count.  Shards start on
    8-row groups (shard_range), so the word ranges concatenate; only the last
    rank may end in a partial group.  Used to check a sharded result against
    one device's scan of all rows (bench.py --gpus N)."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    mine = torch.tensor([n_local], dtype=torch.int64,
                        device="cpu" if dist.get_backend(group) == "gloo" else codes.device)
    ns = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(ns, mine, group=group)
    ns = [int(x.item()) for x in ns]
    if any(n % 8 for n in ns[:-1]):
        raise ValueError(f"shards must hold whole 8-row groups except the last: {ns}")
    words = [-(-n // 8) * m for n in ns]
    wmax = max(max(words), 1)
    pad = torch.zeros(wmax, dtype=torch.int32, device=codes.device)
    pad[:words[rank]] = codes[:words[rank]].view(torch.int32)
    out = torch.empty(world * wmax, dtype=torch.int32, device=codes.device)
    _all_gather_into(out, pad, group)
    whole = torch.cat([out[r * wmax:r * wmax + words[r]] for r in range(world)])
    return whole.view(torch.uint32), sum(ns)


def sharded_topk(codes_shard: torch.Tensor, n_shard: int, qluts: torch.Tensor, k: int, metric,
                 index_base: int, group=None, variant: int = 0) -> torch.Tensor:
    """Top-k over the union of all ranks' shards (every rank gets the result)."""
    from . import topk, topk_merge
    local = topk(codes_shard, n_shard, qluts, k, metric, index_base=index_base, variant=variant)
    if dist.get_world_size(group) == 1:
        return local
    return topk_merge(gather_keys(local, group))


def query_range(nq: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous query slice of `rank` for the query-sharded mode."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    per = -(-nq // world)
    q0 = min(rank * per, nq)
    return q0, min(q0 + per, nq)


def gather_query_slices(local: torch.Tensor, nq: int, group=None) -> torch.Tensor:
    """Each rank's [q1 - q0][k] keys (its query_range slice) -> [nq][k] on every
    rank: one all_gather_into_tensor of equal, padded slices."""
    world = dist.get_world_size(group)
    per = -(-nq // world)
    k = local.shape[1]
    pad = torch.full((per, k), -1, dtype=torch.int64, device=local.device)
    pad[:local.shape[0]] = local.contiguous().view(torch.int64)
    out = torch.empty((world * per, k), dtype=torch.int64, device=local.device)
    _all_gather_into(out, pad, group)
    return out[:nq].view(torch.uint64)


def query_sharded_topk(codes: torch.Tensor, n: int, qluts: torch.Tensor, k: int, metric, group=None,
                       variant: int = 0) -> torch.Tensor:
    """Replicated database, queries split over the ranks: rank r
    scans all n rows for its query slice, so no merge is needed -- the only
    exchange is gathering the disjoint result slices.  Pays off when the codes
    fit on every GPU (c5's 0.8 GB does) and the queries outnumber the ranks."""
    from . import topk
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    q0, q1 = query_range(qluts.shape[0], world, rank)
    local = topk(codes, n, qluts[q0:q1].contiguous(), k, metric, variant=variant) if q1 > q0 else \
        torch.empty((0, k), dtype=torch.uint64, device=codes.device)
    if world == 1:
        return local
    return gather_query_slices(local, qluts.shape[0], group)
