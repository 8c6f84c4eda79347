"""-m gpu parity on the horizons the bench times, in its launch configurations, plus edge
cases driven through the C ABI and the score function itself:

* C5 exactly as bench.py runs it on one GPU: 1024 replicas in the default layout (256-thread
  CTAs, three per SM, each replica's 250-request run replayed as consecutive tasks of a
  persistent grid, so a replica's state moves between SMs inside a launch), 25 launches of
  250 requests per replica (the default 5 warm-up + 20 timed steps); sampled replicas
  replayed by the oracle over all 6 250 requests;
* C3 (balanced, 16 384-block pool, multi-CTA group) over its first 50 000 requests;
* C4 on its full 4M-block pool from the empty pool through 500 eviction rounds past the fill
  (SAE_LONG=1: 11 000 rounds, through the window the bench's C4 workload times -- its pool
  fills at request ~91 K, the timed steps are requests 106 K-112 K);
* C4x: the same trace on a 2^24-block pool, 500 eviction rounds past the fill;
* edge cases the trace generator never produces: equal arrival times, sigma at its 0.1 floor
  with large dt so that P = 0 ties are broken by (last, id), K = 1, one-token prompts with no
  decode, admissions larger than free + unpinned space (k > U);
* Eq.(1)-(3) on the device (sae_priority) bit-equal to the oracle on dense and ulp-adjacent
  dt grids, and non-increasing in dt within every multi-turn class."""
import math
import os
import time

import numpy as np
import pytest
import torch

import oracle
from paper_2605_18825_b200 import configs as C
from paper_2605_18825_b200 import replicas as RP
from paper_2605_18825_b200 import sae as S
from paper_2605_18825_b200 import tracegen as T
from tests.gpu_helpers import assert_stats_equal, assert_traj_equal, compare_replay, u32, unpack
from tests.microtrace import edge_trace as _edge_trace
from tests.test_prop_monotone import dt_grid, param_sets

pytestmark = pytest.mark.gpu


def test_c5_bench_launch_structure():
    per, steps, R = 250, 25, 1024
    n = per * steps
    traces = []
    for sd in range(32):
        t = T.generate(C.get("c5", n_requests=n), seed=0x5AEC1000 + sd)
        T.materialize(t)
        traces.append(t)
    pol = C.policy_config(2304)
    cache = S.SaeCache(2304, n_replicas=R, policy=pol, traj_capacity=256)
    for r in range(R):
        cache.set_params(r, C.c5_point_params(RP.layout(r)[1]))
    lay = cache.layout()
    assert lay["ctas_per_replica"] == 1 and lay["threads"] == 256, lay
    if lay["coresident"] < R:            # (every B200: 148 SMs x 3 < 1024)
        assert lay["chunks"] > 1, lay
    sample = (0, 1, 31, 32, 300, 443, 444, 517, 700, 887, 1022, 1023)
    got = {r: ([], []) for r in sample}
    # one device-resident token arena of the 32 seeds (as bench.py); per step only the
    # request arrays of the 1024 replicas are built
    offs = np.cumsum([0] + [t["n_tokens"] for t in traces]).astype(np.uint64)
    tok_d = torch.from_numpy(np.concatenate([t["tokens"] for t in traces]).view(np.int32)).cuda()
    typ_d = torch.from_numpy(np.concatenate([t["types"] for t in traces])).cuda()
    seed_of = [RP.layout(r)[0] for r in range(R)]
    for s in range(steps):
        sl = slice(s * per, (s + 1) * per)
        cols = {k: [] for k in ("arrival", "prompt_off", "prompt_len", "decode_off", "decode_len",
                                "flags", "spb", "replica")}
        for r in range(R):
            t = traces[seed_of[r]]
            for k in ("arrival", "prompt_len", "decode_len", "flags", "spb"):
                cols[k].append(t[k][sl])
            cols["prompt_off"].append(t["prompt_off"][sl] + offs[seed_of[r]])
            cols["decode_off"].append(t["decode_off"][sl] + offs[seed_of[r]])
            cols["replica"].append(np.full(per, r, np.uint32))
        batch = {k: np.concatenate(v) for k, v in cols.items()}
        batch["n"] = R * per
        batch["tokens"], batch["types"] = np.zeros(1, np.uint32), np.zeros(1, np.uint8)
        b = S.batch_to_torch(batch)
        b["tokens"], b["types"] = tok_d, typ_d
        out = cache.admit_batch(b)
        torch.cuda.synchronize()
        o4, _ = unpack(out, batch["n"])
        vo = out["victim_off"].cpu().numpy()
        vids = u32(out["victim_ids"])
        for r in sample:
            off = r * per
            got[r][0].append(o4[off:off + per])
            got[r][1].extend(int(v) for i in range(per) for v in vids[vo[off + i]:vo[off + i] + o4[off + i, 3]])
    for r in sample:
        sd, pt = RP.layout(r)
        p = dict(pol)
        p["params"] = C.c5_point_params(pt)
        ref = oracle.Replica(p).replay(traces[sd], want_hashes=False)
        assert np.array_equal(np.concatenate(got[r][0]), ref.out4), r
        assert got[r][1] == [int(v) for v in ref.victims], r
        assert_stats_equal(cache.stats(r), ref.stats)
        tj = cache.traj(r)
        assert_traj_equal(tj, ref.traj[len(ref.traj) - len(tj):])


def test_c3_first_50k_requests():
    tr = T.make("c3", n_requests=50_000)
    t0 = time.time()
    compare_replay(tr, C.policy_config(16384), check_hashes=True, traj=1 << 16)
    print("c3 50K parity in %.0f s" % (time.time() - t0))


def _c4_first_rounds(extra):
    tr = T.make("c4", n_requests=100_000 + extra)
    pol = C.policy_config(tr["config"]["capacity"])
    cache = S.SaeCache(pol["capacity"], policy=pol)
    b = S.batch_to_torch(T.single_batch(tr))
    out = cache.admit_batch(b, want_hashes=True)
    torch.cuda.synchronize()
    o4, victims = unpack(out, tr["n"])
    first = int(np.nonzero(o4[:, 3] > 0)[0][0])
    return tr, pol, cache, out, o4, victims, first


@pytest.mark.parametrize("rounds", [500] + ([11000] if os.environ.get("SAE_LONG") else []))
def test_c4_full_pool_through_eviction_rounds(rounds):
    """The empty 4M-block pool filled by the trace (~90K requests), then `rounds` eviction
    rounds; every hash, per-request output and victim id identical to the oracle (its rescans
    threaded over the host cores)."""
    tr, pol, cache, out, o4, victims, first = _c4_first_rounds(rounds + 2000)
    hi = first + rounds
    t0 = time.time()
    R = oracle.Replica(pol)
    ref = R.replay(tr, 0, hi)
    print("c4: pool full at request %d; oracle through %d eviction rounds in %.0f s"
          % (first, rounds, time.time() - t0))
    tb = int(ref.boff[hi])
    assert np.array_equal(out["block_hash"][:tb].cpu().numpy().view(np.uint64), ref.hashes)
    assert np.array_equal(o4[:hi], ref.out4)
    nv = int(ref.voff[hi])
    assert nv > 0 and np.array_equal(victims[:nv], ref.victims)


def test_c4x_pool_500_rounds_past_the_fill():
    """C4x: the C4 trace on a 2^24-block pool (scan records beyond L2, the
    bulk-copy streaming path with evict_first), filled from empty (~0.4 M requests), then 500
    eviction rounds; every hash, per-request output and victim id identical to the oracle."""
    n = 470_000
    tr = T.make("c4", n_requests=n)
    pol = C.policy_config(1 << 24)
    cache = S.SaeCache(pol["capacity"], policy=pol)
    b = S.batch_to_torch(T.single_batch(tr))
    out = cache.admit_batch(b, want_hashes=True)
    torch.cuda.synchronize()
    o4, victims = unpack(out, tr["n"])
    ev = np.nonzero(o4[:, 3] > 0)[0]
    assert len(ev) > 0, "the 2^24-block pool never filled"
    first = int(ev[0])
    hi = min(first + 500, n)
    assert hi - first >= 500, (first, n)
    t0 = time.time()
    ref = oracle.Replica(pol).replay(tr, 0, hi)
    print("c4x: pool full at request %d; oracle through 500 eviction rounds in %.0f s"
          % (first, time.time() - t0))
    tb = int(ref.boff[hi])
    assert np.array_equal(out["block_hash"][:tb].cpu().numpy().view(np.uint64), ref.hashes)
    assert np.array_equal(o4[:hi], ref.out4)
    nv = int(ref.voff[hi])
    assert nv > 0 and np.array_equal(victims[:nv], ref.victims)


# ------------------------------------------------------------------------------------
@pytest.mark.parametrize("case", ["equal_arrivals", "p_zero_ties", "k1", "one_token", "k_gt_u"])
def test_edge_cases_through_the_abi(case):
    p = dict(C.DEFAULT_PARAMS)
    K, cap = 100, 24
    kw = {}
    if case == "equal_arrivals":
        kw = dict(equal_times=True)
    elif case == "p_zero_ties":
        p["mu"], p["sigma"] = [-2.0, -2.0], [0.1, 0.1]   # z > 30 once dt > e^1: P = 0 ties
        p["learn_flags"] = C.L_TOKENS | C.L_QUEUES        # keep sigma at its floor
    elif case == "k1":
        K = 1
    elif case == "one_token":
        kw = dict(one_token=True)
    elif case == "k_gt_u":
        cap = 6
        kw = dict(big_requests=True)
    seed = {"equal_arrivals": 11, "p_zero_ties": 12, "k1": 13, "one_token": 14, "k_gt_u": 15}[case]
    tr = _edge_trace(seed, 400, **kw)
    compare_replay(tr, C.policy_config(cap, K=K, params=p), check_hashes=True)


def test_priority_device_bit_equal_and_monotone():
    for pi, p in enumerate(param_sets()):
        g = dt_grid(pi)
        n = len(g)
        rng = np.random.default_rng(pi)
        for q in (1, 2, 3):
            for tau in range(4):
                omax = rng.integers(1, 60, n).astype(np.uint32)
                ob = (rng.integers(0, 1 << 30, n) % (omax + 1)).astype(np.uint32)
                dev = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a).view(dt)).cuda()
                P = S.priority(p, dev(np.full(n, q, np.uint8), np.uint8), dev(np.full(n, tau, np.uint8), np.uint8),
                               dev(g, np.float64), dev(ob, np.int32), dev(omax, np.int32)).cpu().numpy()
                ref = np.array([oracle.priority(p, q, tau, float(x), int(b), int(m))
                                for x, b, m in zip(g, ob, omax)])
                assert np.array_equal(P.view(np.uint64), ref.view(np.uint64)), (pi, q, tau)
                if q < 3:
                    assert np.all(P[1:] <= P[:-1]), (pi, q, tau)
