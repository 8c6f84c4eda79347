"""Property tests over random micro-traces (hypothesis; SURVEY §4 tests/prop): small traces over
a shared block vocabulary (prefix reuse, orphans, ghost hits, partial and decode blocks, every
flag combination, equal arrival times, requests larger than the pool), random capacities,
learner periods K and learners on/off.

* oracle (-m "not gpu"): after every request the pool never exceeds C; hits + misses = the
  request's blocks; every hit's block was resident before the request (strict prefix);
  every victim was an unpinned resident; Stage 1 first: EF victims lead, in (ntok, id) order
  (Alg.1 Evict); with a pool larger than the whole trace nothing is evicted and the
  hits of a request are exactly the longest prefix of its block chain seen in earlier
  requests (brute force).
* GPU (-m gpu): the same traces through the C ABI equal the oracle bit for bit."""
import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import oracle
from paper_2605_18825_b200 import configs as C
from tests.microtrace import edge_trace

B = 16
TRACES = st.tuples(st.integers(0, 2 ** 31 - 1), st.integers(4, 60), st.booleans(), st.booleans(),
                   st.booleans())


def _policy(cap, K, learn):
    p = dict(C.DEFAULT_PARAMS)
    if not learn:
        p["learn_flags"] = 0
    return C.policy_config(cap, K=K, params=p)


def _requests(tr):
    for i in range(tr["n"]):
        po, pl = int(tr["prompt_off"][i]), int(tr["prompt_len"][i])
        do, dl = int(tr["decode_off"][i]), int(tr["decode_len"][i])
        yield (tr["arrival"][i], tr["tokens"][po:po + pl], tr["types"][po:po + pl],
               tr["tokens"][do:do + dl], tr["flags"][i], tr["spb"][i], pl, dl)


@settings(max_examples=60, deadline=None)
@given(spec=TRACES, cap=st.sampled_from([3, 4, 6, 9, 16, 40]), K=st.sampled_from([1, 2, 5, 100]),
       learn=st.booleans())
def test_oracle_invariants_on_random_traces(spec, cap, K, learn):
    seed, n, one_tok, eq, big = spec
    tr = edge_trace(seed, n, one_token=one_tok, equal_times=eq, big_requests=big)
    R = oracle.Replica(_policy(cap, K, learn))
    for now, pt, py, dt, fl, spb, pl, dl in _requests(tr):
        before = R.resident()
        by_hash = {int(h): (int(q), int(nt), int(bid)) for h, q, nt, bid in
                   zip(before["hash"], before["q"], before["ntok"], before["id"])}
        rc, res, vic, H, tau = R.admit_req(now, pt, py, dt, fl, spb)
        assert rc == 0
        nb = len(H)
        assert nb == -(-pl // B) + -(-dl // B)
        assert int(res[0]) + int(res[1]) == nb
        st_ = R.stats()
        assert st_.resident <= cap
        for j in range(int(res[0])):                     # strict prefix of resident blocks
            assert int(H[j]) in by_hash
        pin = {int(h) for h in H if int(h) in by_hash}
        pinned_ids = {by_hash[h][2] for h in pin}
        id2 = {bid: (q, nt) for _, (q, nt, bid) in by_hash.items()}
        for v in vic:                                     # victims: unpinned residents
            assert int(v) in id2 and int(v) not in pinned_ids
        ef = sorted((nt, bid) for hsh, (q, nt, bid) in by_hash.items() if q == 0 and hsh not in pin)
        e = min(len(vic), len(ef))
        assert [int(v) for v in vic[:e]] == [bid for _, bid in ef[:e]]   # Stage 1 first
        for v in vic[e:]:
            assert id2[int(v)][0] != 0


@settings(max_examples=40, deadline=None)
@given(spec=TRACES, learn=st.booleans())
def test_unbounded_pool_hits_are_longest_seen_prefix(spec, learn):
    seed, n, one_tok, eq, big = spec
    tr = edge_trace(seed, n, one_token=one_tok, equal_times=eq, big_requests=big)
    total = int((-(-tr["prompt_len"].astype(np.int64) // B) - (-tr["decode_len"].astype(np.int64) // B)).sum())
    R = oracle.Replica(_policy(total + 1, 100, learn))
    seen = set()
    for now, pt, py, dt, fl, spb, pl, dl in _requests(tr):
        rc, res, vic, H, tau = R.admit_req(now, pt, py, dt, fl, spb)
        assert rc == 0 and len(vic) == 0
        h = 0
        while h < len(H) and int(H[h]) in seen:
            h += 1
        assert int(res[0]) == h
        seen.update(int(x) for x in H)


@pytest.mark.gpu
@settings(max_examples=25, deadline=None)
@given(spec=TRACES, cap=st.sampled_from([3, 6, 16, 40]), K=st.sampled_from([1, 3, 100]),
       learn=st.booleans())
def test_random_traces_gpu_equal_oracle(spec, cap, K, learn):
    from tests.gpu_helpers import compare_replay
    seed, n, one_tok, eq, big = spec
    tr = edge_trace(seed, n, one_token=one_tok, equal_times=eq, big_requests=big)
    compare_replay(tr, _policy(cap, K, learn), check_hashes=True)
