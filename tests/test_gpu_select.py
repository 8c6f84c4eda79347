"""-m gpu: sae_select, the fused score/select pass alone (K3; Alg.1 Evict's choice),
is read-only and chooses exactly the victims the oracle's Evict takes next: private pools
(one CTA) and a multi-CTA replica group, several passes per launch, m up to 96."""
import numpy as np
import pytest

import oracle
from paper_2605_18825_b200 import configs as C
from paper_2605_18825_b200 import sae as S
from paper_2605_18825_b200 import tracegen as T
from tests.gpu_helpers import assert_stats_equal, gpu_replay, u32

pytestmark = pytest.mark.gpu


def _check_select(tr, pol, hi, ctas, ms):
    cache, b, out = gpu_replay(tr, pol, hi=hi, ctas=ctas)
    R = oracle.Replica(pol)
    R.replay(tr, 0, hi)
    now = float(tr["arrival"][hi - 1]) + 2.0
    st0 = cache.stats(0)
    for m in ms:
        for passes in (1, 3):
            ids, n = cache.select(0, m, now, passes=passes)
            cache.sync()
            got = list(u32(ids)[:int(n.item())])
            # the oracle's next m victims (Evict x m at `now`), taken on a copy of its state:
            # no learner may fire inside them (keys are frozen between firings, A14)
            E = R.stats().E
            mm = min(m, pol["K"] - E % pol["K"])
            R2 = oracle.Replica(pol)
            R2.replay(tr, 0, hi)
            rc, ref = R2.evict(mm, now)
            assert rc == 0 and got[:mm] == list(ref)
            assert len(got) == min(m, st0.resident)
    # read-only: every counter, parameter and the clock unchanged
    assert_stats_equal(cache.stats(0), R.stats())
    # and the next real eviction takes the same blocks
    E = R.stats().E
    k = min(40, pol["K"] - E % pol["K"])
    ids_s, _ = cache.select(0, k, now)
    ids_e, n_e = cache.evict(0, k, now)
    assert list(u32(ids_s)[:k]) == list(u32(ids_e)[:int(n_e.item())])


def test_select_private_pool():
    tr = T.make("c2", n_requests=1500)
    _check_select(tr, C.policy_config(2304, K=100), 1500, 0, (1, 17, 96))


def test_select_group_pool():
    tr = T.generate(C.get("c4", n_requests=2500, n_tpl={"tool_use": 1 << 10, "programming": 1 << 8},
                          seed=0x5AEC4444))
    T.materialize(tr)
    _check_select(tr, C.policy_config(6000, K=100), 1500, 4, (5, 96))


def test_select_rejects_bad_arguments():
    tr = T.make("c1")
    cache, b, out = gpu_replay(tr, C.policy_config(64, K=8), hi=50)
    with pytest.raises(S.SaeError):
        cache.select(0, 97, 1e9)
    with pytest.raises(S.SaeError):
        cache.select(0, 4, 1e9, passes=0)
    cache.select(0, 4, 0.0)           # earlier than the replica's clock: sticky SAE_E_TIME
    with pytest.raises(S.SaeError) as e:
        cache.sync()
    assert e.value.status == -5
