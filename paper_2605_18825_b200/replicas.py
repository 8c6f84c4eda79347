"""C5 replica sharding and the optional mean_w sync.

Replica r (global index, 0..R_total-1) replays seed ``r // n_points`` at parameter point
``r % n_points``.  GPU g of G owns the contiguous replicas [g*R/G, (g+1)*R/G); there is no
data-path collective.  The optional ``mean_w@E`` mode, every E requests per replica,
all-gathers the fp64 parameter records (NCCL over NVLink) and replaces each replica's
token-type weights by the fixed-order mean over the seeds of its point
(``sae_params_point_mean``), so results do not depend on the GPU count.
"""
from __future__ import annotations

import ctypes


def shard(n_total: int, world: int, rank: int) -> tuple[int, int]:
    return n_total * rank // world, n_total * (rank + 1) // world


def layout(r: int, n_points: int = 32) -> tuple[int, int]:
    """(seed index, parameter point) of global replica r."""
    return r // n_points, r % n_points


def gather_params(local, group=None):
    """All-gather [R_local, P] float64 parameter records into [R_total, P] in global replica
    order (rank-major == contiguous shards).  Shards may differ in size by one (shard()):
    every rank pads to the largest and the padding is dropped after the gather."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return local
    ws = dist.get_world_size(group)
    n = torch.tensor([local.shape[0]], dtype=torch.int64, device=local.device)
    sizes = [torch.zeros_like(n) for _ in range(ws)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(x.item()) for x in sizes]
    pad = torch.zeros((max(sizes),) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(ws)]
    dist.all_gather(parts, pad.contiguous(), group=group)
    return torch.cat([p[:k] for p, k in zip(parts, sizes)], 0)


def sync_mean_w(cache, n_points: int = 32, group=None, stream=None):
    """mean_w sync of one sae_ctx holding this rank's contiguous shard of replicas: all-gather
    the parameter records, fixed-order mean of w over the seeds of each point (identical at
    any GPU count), scatter this rank's shard back."""
    import torch.distributed as dist
    from . import sae as S
    local = cache.params_gather(stream=stream)
    allp = gather_params(local, group)
    mean = S.params_point_mean(allp, n_points, stream=stream)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        lo, hi = shard(allp.shape[0], dist.get_world_size(group), dist.get_rank(group))
    else:
        lo, hi = 0, allp.shape[0]
    cache.params_scatter(mean[lo:hi].contiguous(), stream=stream)


def allreduce_counters(cache, group=None, stream=None):
    """Job-wide totals of the additive hit / eviction / miss-after-evict counters: the device
    sums this ctx's replicas (sae_counters_device), then an int64 SUM all-reduce (NCCL over
    NVLink; exact in any order).  Returns {field: total} on every rank."""
    import torch.distributed as dist
    from . import sae as S
    t = cache.counters_device(stream=stream)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return dict(zip(S.COUNTER_FIELDS, (int(x) for x in t.cpu().tolist())))
