"""-m gpu: the baseline / ablation modes (include/sae.h SAE_MODE_*)
replayed by the kernels, bit-exact against the oracle: LRU, LFU and Token-Weight-Only on C1
and on a C2 prefix, and a mixed sweep (every variant of paper_2605_18825_b200.ablation as a
replica of one ctx, as scripts/ablation.py runs them)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2605_18825_b200 import ablation as A
from paper_2605_18825_b200 import configs as C
from paper_2605_18825_b200 import sae as S
from paper_2605_18825_b200 import tracegen as T
from tests.gpu_helpers import assert_stats_equal, assert_traj_equal, compare_replay, u32, unpack

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", [C.MODE_LRU, C.MODE_LFU, C.MODE_TWO])
def test_baseline_mode_c1(mode):
    p = dict(C.DEFAULT_PARAMS, mode=mode)
    compare_replay(T.make("c1"), C.policy_config(64, K=8, params=p))


@pytest.mark.parametrize("mode", [C.MODE_LRU, C.MODE_LFU, C.MODE_TWO])
def test_baseline_mode_c2_prefix(mode):
    p = dict(C.DEFAULT_PARAMS, mode=mode)
    compare_replay(T.make("c2", n_requests=4000), C.policy_config(2304, params=p))


def test_ablation_variants_side_by_side():
    tr = T.make("c5", n_requests=3000)
    var = A.variants()
    names = sorted(var)
    R = len(names)
    pol = C.policy_config(2304)
    cache = S.SaeCache(2304, n_replicas=R, policy=pol, traj_capacity=1 << 12)
    for r, nm in enumerate(names):
        cache.set_params(r, var[nm])
    batch = T.replicate([tr], [0] * R)
    out = cache.admit_batch(S.batch_to_torch(batch))
    torch.cuda.synchronize()
    o4, _ = unpack(out, batch["n"])
    vo = out["victim_off"].cpu().numpy()
    vids = u32(out["victim_ids"])
    n = tr["n"]
    for r, nm in enumerate(names):
        p = dict(pol)
        p["params"] = var[nm]
        ref = oracle.Replica(p).replay(tr, want_hashes=False)
        off = r * n
        assert np.array_equal(o4[off:off + n], ref.out4), nm
        got = np.concatenate([vids[vo[off + i]:vo[off + i] + o4[off + i, 3]] for i in range(n)])
        assert np.array_equal(got, ref.victims), nm
        assert_stats_equal(cache.stats(r), ref.stats)
        assert_traj_equal(cache.traj(r), ref.traj)
