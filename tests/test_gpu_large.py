"""-m gpu parity for pools larger than one CTA's candidate buffer (C > 4096): the
global candidate buffer, the group-parallel radix narrowing and multi-CTA replica
groups (cooperative launch), against the oracle, bit-exact."""
import numpy as np
import pytest
import torch

import oracle
from paper_2605_18825_b200 import configs as C
from paper_2605_18825_b200 import sae as S
from paper_2605_18825_b200 import tracegen as T
from tests.gpu_helpers import assert_stats_equal, assert_traj_equal, compare_replay, u32, unpack

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def st_trace():
    tr = T.generate(C.get("c4", n_requests=2500, n_tpl={"tool_use": 1 << 10, "programming": 1 << 8},
                          seed=0x5AEC4444))
    T.materialize(tr)
    return tr


@pytest.fixture(scope="module")
def bal_trace():
    tr = T.generate(C.get("c3", n_requests=2000, seed=0x5AEC3333))
    T.materialize(tr)
    return tr


@pytest.mark.parametrize("ctas", [1, 2, 4])
def test_large_pool_single_trace(st_trace, ctas):
    compare_replay(st_trace, C.policy_config(6000, K=100), ctas=ctas)


def test_c3_shaped_pool_auto_group(bal_trace):
    compare_replay(bal_trace, C.policy_config(16384, K=100))


def test_large_pool_small_K_many_firings(bal_trace):
    compare_replay(bal_trace, C.policy_config(5000, K=7), ctas=3)


def test_large_pool_learner_variants(st_trace):
    p = dict(C.DEFAULT_PARAMS)
    p["learn_flags"] = C.L_DEFAULT | C.L_QUEUE_RELATIVE
    compare_replay(st_trace, C.policy_config(4500, K=50, params=p), ctas=2)


def test_large_pool_multi_replica_groups(st_trace, bal_trace):
    traces = [st_trace, bal_trace]
    R = 3
    rep_of = [0, 1, 0]
    batch = T.replicate(traces, rep_of)
    pol = C.policy_config(4500, K=60)
    cache = S.SaeCache(4500, n_replicas=R, policy=pol, traj_capacity=1 << 14, ctas_per_replica=2)
    pts = [0, 17, 31]
    for r in range(R):
        cache.set_params(r, C.c5_point_params(pts[r]))
    out = cache.admit_batch(S.batch_to_torch(batch))
    torch.cuda.synchronize()
    o4, _ = unpack(out, batch["n"])
    vo = out["victim_off"].cpu().numpy()
    vids = u32(out["victim_ids"])
    off = 0
    for r in range(R):
        tr = traces[rep_of[r]]
        p = dict(pol)
        p["params"] = C.c5_point_params(pts[r])
        ref = oracle.Replica(p).replay(tr)
        n = tr["n"]
        assert np.array_equal(o4[off:off + n], ref.out4), r
        got = np.concatenate([vids[vo[off + i]:vo[off + i] + o4[off + i, 3]] for i in range(n)])
        assert np.array_equal(got, ref.victims), r
        assert_stats_equal(cache.stats(r), ref.stats)
        assert_traj_equal(cache.traj(r), ref.traj)
        off += n


def test_large_pool_evict_update(st_trace):
    pol = C.policy_config(6000, K=100)
    from tests.gpu_helpers import gpu_replay, assert_params_equal
    cache, b, out = gpu_replay(st_trace, pol, hi=1500, ctas=4)
    R = oracle.Replica(pol)
    R.replay(st_trace, 0, 1500)
    now = float(st_trace["arrival"][1499]) + 3.0
    for k in (250, 7, 400):
        ids, n = cache.evict(0, k, now)
        rc, ref = R.evict(k, now)
        assert int(n.item()) == len(ref)
        assert list(u32(ids)[:len(ref)]) == list(ref)
        now += 1.5
    cache.update(0)
    R.update()
    st = cache.stats(0)
    assert_params_equal(S.params_dict(st.params), R.params())
    assert_stats_equal(st, R.stats())
