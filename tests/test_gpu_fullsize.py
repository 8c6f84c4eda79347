"""-m gpu parity at BASELINE.json's full C4 size, in the launch configuration bench
uses (4M-block pool, one 148-CTA cooperative group): the oracle replays the trace prefix
up to 15 rounds past the first eviction (the pool fills after ~90K requests) and every
block hash, per-request output and victim id of that prefix must be identical."""
import time

import numpy as np
import pytest
import torch

import oracle
from paper_2605_18825_b200 import configs as C
from paper_2605_18825_b200 import sae as S
from paper_2605_18825_b200 import tracegen as T
from tests.gpu_helpers import u32, unpack

pytestmark = pytest.mark.gpu


def test_c4_full_pool_first_eviction_rounds():
    n = 100_000
    tr = T.make("c4", n_requests=n)
    pol = C.policy_config(tr["config"]["capacity"])
    cache = S.SaeCache(pol["capacity"], policy=pol)
    sub = T.single_batch(tr)
    b = S.batch_to_torch(sub)
    out = cache.admit_batch(b, want_hashes=True)
    torch.cuda.synchronize()
    o4, victims = unpack(out, n)
    first = int(np.nonzero(o4[:, 3] > 0)[0][0])
    hi = first + 15
    t0 = time.time()
    R = oracle.Replica(pol)
    ref = R.replay(tr, 0, hi)
    print("oracle prefix of %d requests (%d evicting) in %.1fs" % (hi, 15, time.time() - t0))
    tb = int(ref.boff[hi])
    assert np.array_equal(out["block_hash"][:tb].cpu().numpy().view(np.uint64), ref.hashes)
    assert np.array_equal(o4[:hi], ref.out4)
    nv = int(ref.voff[hi])
    assert nv > 0
    assert np.array_equal(victims[:nv], ref.victims)
    # properties that hold at any size for the rest of the GPU run
    assert np.all(o4[:, 0] + o4[:, 1] == (-(-tr["prompt_len"].astype(np.int64) // 16)
                                          - (-tr["decode_len"].astype(np.int64) // 16)))
    st = cache.stats(0)
    assert st.resident == pol["capacity"]
    assert st.evictions == int(o4[:, 3].sum())
    assert sum(st.resident_by_queue) == st.resident


def test_c2_full_trace_bit_exact():
    """C2 at its full size (100K requests, C=2304), one replica: every output identical."""
    from tests.gpu_helpers import compare_replay
    tr = T.make("c2")
    compare_replay(tr, C.policy_config(2304), check_hashes=True, traj=1 << 17)


def test_c5_full_config_sampled_replicas():
    """C5 exactly as bench.py runs it on one GPU (1024 replicas x 10K requests, C=2304,
    the 256-thread two-CTAs-per-SM variant); sampled replicas replayed by the oracle."""
    from paper_2605_18825_b200 import replicas as RP
    n = 10_000
    traces = []
    for sd in range(32):
        t = T.generate(C.get("c5", n_requests=n), seed=0x5AEC1000 + sd)
        T.materialize(t)
        traces.append(t)
    R = 1024
    pol = C.policy_config(2304)
    cache = S.SaeCache(2304, n_replicas=R, policy=pol)
    for r in range(R):
        cache.set_params(r, C.c5_point_params(RP.layout(r)[1]))
    batch = T.replicate(traces, [RP.layout(r)[0] for r in range(R)])
    out = cache.admit_batch(S.batch_to_torch(batch))
    torch.cuda.synchronize()
    o4, _ = unpack(out, batch["n"])
    vo = out["victim_off"].cpu().numpy()
    vids = u32(out["victim_ids"])
    for r in (0, 31, 32, 517, 1023):
        sd, pt = RP.layout(r)
        p = dict(pol)
        p["params"] = C.c5_point_params(pt)
        ref = oracle.Replica(p).replay(traces[sd], want_hashes=False)
        off = r * n
        assert np.array_equal(o4[off:off + n], ref.out4), r
        got = np.concatenate([vids[vo[off + i]:vo[off + i] + o4[off + i, 3]] for i in range(n)])
        assert np.array_equal(got, ref.victims), r


def test_c3_pool_multi_cta_first_rounds():
    """C3's 16384-block pool (multi-CTA group, as configured by default) on the C3 trace's
    first 3000 requests (the pool fills after ~300)."""
    from tests.gpu_helpers import compare_replay
    tr = T.make("c3", n_requests=3000)
    compare_replay(tr, C.policy_config(16384), check_hashes=True)
