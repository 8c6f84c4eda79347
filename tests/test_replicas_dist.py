"""Multi-process (gloo, world_size 2, CPU) tests of the C5 sharding / parameter-gather host
logic that the NCCL path uses on GPUs."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_18825_b200 import replicas as RP

ND = 21   # sae_params as float64 words


def test_shard_partition_is_disjoint_and_covering():
    for R in (1, 7, 1024, 1025):
        for W in (1, 2, 3, 4, 8):
            seen = []
            for g in range(W):
                lo, hi = RP.shard(R, W, g)
                seen.extend(range(lo, hi))
            assert seen == list(range(R))


def test_layout_seed_point():
    assert RP.layout(0) == (0, 0)
    assert RP.layout(33) == (1, 1)
    assert RP.layout(1023) == (31, 31)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, R, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = RP.shard(R, world, rank)
    local = torch.zeros((hi - lo, ND), dtype=torch.float64)
    for i, r in enumerate(range(lo, hi)):
        rng = np.random.default_rng(r)
        local[i, :5] = torch.from_numpy(rng.uniform(0.1, 5.0, 5))
        local[i, 5] = r
    allp = RP.gather_params(local)
    q.put((rank, allp.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


def test_gather_params_gloo_world2_global_order():
    R, world = 64, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, R, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a0, a1 = res[0], res[1]
    assert np.array_equal(a0, a1)                          # every rank sees the same table
    assert list(a0[:, 5].astype(int)) == list(range(R))    # in global replica order
    # the fixed-order mean is then identical to the single-process computation
    import oracle
    params = [{"w": list(a0[r, :5])} for r in range(R)]
    m = oracle.point_mean_w(params, 32)
    for r in range(R):
        p = r % 32
        exp = [(a0[p, t] + a0[p + 32, t]) / 2.0 for t in range(5)]
        assert m[r]["w"] == exp


class _FakeCache:
    """CPU stand-in of SaeCache for the host logic of sync_mean_w / allreduce_counters
    (params_gather / params_scatter / counters_device): the collectives are real (gloo)."""

    def __init__(self, lo, hi):
        self.lo, self.hi = lo, hi
        self.p = torch.zeros((hi - lo, ND), dtype=torch.float64)
        for i, r in enumerate(range(lo, hi)):
            rng = np.random.default_rng(1000 + r)
            self.p[i, :5] = torch.from_numpy(rng.uniform(0.1, 5.0, 5))
            self.p[i, 5] = r
        self.scattered = None

    def params_gather(self, stream=None):
        return self.p.clone()

    def params_scatter(self, t, stream=None):
        self.scattered = t.clone()

    def counters_device(self, stream=None):
        from paper_2605_18825_b200 import sae as S
        t = torch.zeros(len(S.COUNTER_FIELDS), dtype=torch.int64)
        t[0] = self.hi - self.lo          # "requests": one per local replica
        t[2] = 3 * (self.hi - self.lo)    # "hit_blocks"
        t[5] = (1 << 40) + self.lo        # "evictions": exceeds 32 bits (int64 all-reduce)
        return t


def _point_mean_plain(allp, n_points):
    """Fixed-order mean over seeds (the oracle's order, written out here for the fake)."""
    out = allp.clone()
    S = allp.shape[0] // n_points
    for p in range(n_points):
        for t in range(5):
            s = 0.0
            for i in range(S):
                s = s + float(allp[p + n_points * i, t])
            for i in range(S):
                out[p + n_points * i, t] = s / float(S)
    return out


def _sync_worker(rank, world, port, R, n_points, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_18825_b200 import sae as S
    S.params_point_mean = lambda allp, n, stream=None: _point_mean_plain(allp, n)
    lo, hi = RP.shard(R, world, rank)
    cache = _FakeCache(lo, hi)
    RP.sync_mean_w(cache, n_points=n_points)
    tot = RP.allreduce_counters(cache)
    q.put((rank, lo, hi, cache.scattered.numpy().copy(), tot))
    dist.barrier()
    dist.destroy_process_group()


def test_sync_mean_w_unequal_shards_gloo_world2():
    """R = 65 over 2 ranks (shards of 32 and 33): the padded all-gather, the fixed-order mean
    over the 5 seeds of each of 13 points, the scatter of each rank's own shard, and the int64
    all-reduce of the counters."""
    R, world, n_points = 65, 2, 13
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sync_worker, args=(r, world, port, R, n_points, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, lo, hi, sc, tot = q.get(timeout=120)
        res[rank] = (lo, hi, sc, tot)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = np.concatenate([_FakeCache(*RP.shard(R, world, g)).p.numpy() for g in range(world)])
    ref = _point_mean_plain(torch.from_numpy(full), n_points).numpy()
    for rank, (lo, hi, sc, tot) in res.items():
        assert sc.shape[0] == hi - lo
        assert np.array_equal(sc, ref[lo:hi])
        assert tot["requests"] == R and tot["hit_blocks"] == 3 * R
        assert tot["evictions"] == 2 * (1 << 40) + sum(RP.shard(R, world, g)[0] for g in range(world))
