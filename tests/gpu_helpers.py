"""Shared helpers for the -m gpu parity tests: run the CUDA path through the C ABI
and the oracle on the same seeded inputs and compare element by element."""
from __future__ import annotations

import numpy as np
import torch

import oracle
from paper_2605_18825_b200 import configs as C
from paper_2605_18825_b200 import sae as S
from paper_2605_18825_b200 import tracegen as T


def u32(t):
    return t.cpu().numpy().view(np.uint32)


def gpu_replay(tr, pol, n_replicas=1, traj=1 << 16, lo=0, hi=None, cache=None, ctas=0):
    """Replay requests [lo, hi) of a single-replica trace on the GPU (replica 0)."""
    hi = tr["n"] if hi is None else hi
    sub = {k: tr[k][lo:hi] for k in ("arrival", "prompt_off", "prompt_len", "decode_off",
                                     "decode_len", "flags", "spb")}
    sub["tokens"], sub["types"], sub["n"] = tr["tokens"], tr["types"], hi - lo
    sub["replica"] = np.zeros(hi - lo, np.uint32)
    cache = cache or S.SaeCache(pol["capacity"], n_replicas=n_replicas, policy=pol,
                                traj_capacity=traj, ctas_per_replica=ctas)
    b = S.batch_to_torch(sub)
    out = cache.admit_batch(b, want_hashes=True)
    torch.cuda.synchronize()
    return cache, b, out


def unpack(out, n):
    o4 = np.stack([u32(out[k]) for k in ("hit_blocks", "miss_blocks", "matched_tokens",
                                         "n_victims")], 1)
    vo = out["victim_off"].cpu().numpy()
    vids = u32(out["victim_ids"])
    victims = np.concatenate([vids[vo[i]:vo[i] + o4[i, 3]] for i in range(n)]) if n else np.zeros(0)
    return o4, victims


def assert_params_equal(a: dict, b: dict):
    for k in ("w", "alpha", "mu", "sigma"):
        assert list(a[k]) == list(b[k]), (k, a[k], b[k])
    assert a["gamma"] == b["gamma"]


def assert_traj_equal(tg, tr_):
    assert len(tg) == len(tr_), (len(tg), len(tr_))
    for i, (a, r) in enumerate(zip(tg, tr_)):
        assert a.E == r.E and a.request == r.request, i
        for k in ("w", "alpha", "mu", "sigma"):
            assert list(getattr(a, k)) == list(getattr(r, k)), (i, k, list(getattr(a, k)),
                                                                list(getattr(r, k)))
        assert a.gamma == r.gamma, i


def assert_stats_equal(g, o):
    for k in ("requests", "blocks_looked_up", "hit_blocks", "hit_tokens", "prompt_tokens",
              "evictions", "learner_firings", "eviction_rounds", "blocks_scored", "resident",
              "E", "next_id", "gseq"):
        assert getattr(g, k) == getattr(o, k), (k, getattr(g, k), getattr(o, k))
    for k in ("evict_by_queue", "evict_by_type", "mae_by_type", "resident_by_queue", "ts_ev",
              "ts_mae", "ts_hit", "ts_acc", "qh", "qe", "pb_hit", "pb_acc", "iv_len"):
        assert list(getattr(g, k)) == list(getattr(o, k)), (k, list(getattr(g, k)),
                                                            list(getattr(o, k)))


def compare_replay(tr, pol, lo=0, hi=None, check_hashes=True, ctas=0, traj=1 << 16):
    cache, b, out = gpu_replay(tr, pol, lo=lo, hi=hi, ctas=ctas, traj=traj)
    R = oracle.Replica(pol)
    ref = R.replay(tr, lo, hi)
    n = (tr["n"] if hi is None else hi) - lo
    o4, victims = unpack(out, n)
    if check_hashes:
        tb = b["total_blocks"]
        assert np.array_equal(out["block_hash"][:tb].cpu().numpy().view(np.uint64), ref.hashes)
        assert np.array_equal(out["block_tau"][:tb].cpu().numpy(), ref.taus)
    bad = np.nonzero((o4 != ref.out4).any(1))[0]
    assert len(bad) == 0, ("first differing request", int(bad[0]), o4[bad[0]], ref.out4[bad[0]])
    if not np.array_equal(victims, ref.victims):
        i = int(np.nonzero(victims != ref.victims)[0][0])
        raise AssertionError("victim sequence differs at %d: gpu %s oracle %s" %
                             (i, victims[i:i + 8], ref.victims[i:i + 8]))
    st = cache.stats(0)
    assert_stats_equal(st, ref.stats)
    assert_traj_equal(cache.traj(0), ref.traj)
    assert_params_equal(S.params_dict(st.params), R.params())
    return cache, R, ref
