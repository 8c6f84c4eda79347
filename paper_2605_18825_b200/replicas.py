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
    order (rank-major == contiguous shards)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return local
    ws = dist.get_world_size(group)
    parts = [torch.empty_like(local) for _ in range(ws)]
    dist.all_gather(parts, local.contiguous(), group=group)
    return torch.cat(parts, 0)


def sync_mean_w(cache, n_points: int = 32, group=None, stream=None):
    """mean_w sync of one sae_ctx holding this rank's contiguous shard of replicas."""
    import torch
    import torch.distributed as dist
    from . import sae as S
    local = cache.params_gather(stream=stream)
    allp = gather_params(local, group)
    mean = S.params_point_mean(allp, n_points, stream=stream)
    if dist.is_initialized() and dist.get_world_size() > 1:
        lo, hi = shard(allp.shape[0], dist.get_world_size(), dist.get_rank())
    else:
        lo, hi = 0, allp.shape[0]
    cache.params_scatter(mean[lo:hi].contiguous(), stream=stream)
