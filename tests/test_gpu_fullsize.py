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
