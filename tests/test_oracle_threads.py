"""The oracle's threaded key computation for large pools (C4's scan split across
the host cores) gives exactly the serial rescan's victims: the m smallest keys under a total
order do not depend on how the pool is partitioned."""
import os

import numpy as np

import oracle
from paper_2605_18825_b200 import configs as C
from paper_2605_18825_b200 import tracegen as T


def _replay(tr, pol, threads):
    old = os.environ.get("ORACLE_THREADS")
    os.environ["ORACLE_THREADS"] = str(threads)
    try:
        return oracle.Replica(pol).replay(tr, want_hashes=False)
    finally:
        if old is None:
            del os.environ["ORACLE_THREADS"]
        else:
            os.environ["ORACLE_THREADS"] = old


def test_threaded_scan_equals_serial():
    tr = T.make("c4", n_requests=1350, capacity=65536)
    pol = C.policy_config(65536, K=16)
    a = _replay(tr, pol, 1)
    b = _replay(tr, pol, 5)
    assert int(a.stats.evictions) > 100 and int(a.stats.learner_firings) > 5
    assert np.array_equal(a.out4, b.out4)
    assert np.array_equal(a.victims, b.victims)
    assert [list(t.w) for t in a.traj] == [list(t.w) for t in b.traj]
