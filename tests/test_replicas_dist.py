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
