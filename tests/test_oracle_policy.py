"""Policy pins for the oracle (SURVEY c.7): LRU recovery, brute-force OPT bound,
capacity / partition / stage-order invariants, hand-traced evictions, errors."""
import itertools

import numpy as np
import pytest

import oracle
from paper_2605_18825_b200 import configs as C
from paper_2605_18825_b200 import tracegen as T
from tests.test_oracle_hash import chain_ref


def replica(cap, K=100, **pover):
    p = dict(C.DEFAULT_PARAMS)
    p.update(pover)
    return oracle.Replica(C.policy_config(cap, K=K, params=p))


# ------------------------------------------------------------------------------------
class LRU:
    """Textbook LRU (evict min (last, id)) with the replay's admission semantics
    (pinning of the request's resident blocks, orphan refresh, overflow cap)."""

    def __init__(self, cap):
        self.cap, self.res, self.next_id = cap, {}, 0

    def admit(self, now, chain):
        h = 0
        while h < len(chain) and chain[h] in self.res:
            h += 1
        pin = {x for x in chain if x in self.res}
        for x in pin:
            self.res[x][0] = now
        new = [x for x in chain[h:] if x not in self.res]
        f = self.cap - len(self.res)
        U = len(self.res) - len(pin)
        k = max(0, len(new) - f)
        if k > U:
            k, new = U, new[: f + U]
        cand = sorted((v[0], v[1], x) for x, v in self.res.items() if x not in pin)
        victims = []
        for last, bid, x in cand[:k]:
            victims.append(bid)
            del self.res[x]
        for x in new:
            self.res[x] = [now, self.next_id]
            self.next_id += 1
        return h, victims


def test_lru_recovered_when_weights_uniform_and_learner_off():
    """north_star: 'LRU is recovered when the semantic weights are uniform and the
    learner is disabled' -- holds when every block sits in one multi-turn queue
    (SURVEY Appendix B): all requests multi-turn chat, no CoT, no decode."""
    rng = np.random.default_rng(21)
    for trial in range(8):
        R = replica(48, w=[1.0] * 5, alpha=[1.0] * 3, learn_flags=0)
        L = LRU(48)
        pool = [rng.integers(0, 1 << 17, 16 * int(rng.integers(1, 6))).astype(np.uint32)
                for _ in range(10)]
        now = 0.0
        for step in range(150):
            toks = np.concatenate([pool[i] for i in rng.integers(0, 10, rng.integers(1, 4))])
            toks = toks[: len(toks) - int(rng.integers(0, 9))]
            now += float(rng.exponential(5.0)) + 1e-6
            rc, res, vic, H, tau = R.admit_req(now, toks, np.ones(len(toks), np.uint8), [],
                                               1 | 4, 0)
            assert rc == 0
            h, lv = L.admit(now, chain_ref(toks))
            assert res[0] == h
            assert list(vic) == lv, (trial, step)


def _opt_hits(cap, chains):
    """Exhaustive best total hit blocks over all victim choices (same admission rules)."""
    from functools import lru_cache

    @lru_cache(maxsize=None)
    def go(i, res):
        if i == len(chains):
            return 0
        chain = chains[i]
        resd = set(res)
        h = 0
        while h < len(chain) and chain[h] in resd:
            h += 1
        pin = {x for x in chain if x in resd}
        new = []
        for x in chain[h:]:
            if x not in resd and x not in new:
                new.append(x)
        f = cap - len(resd)
        U = sorted(resd - pin)
        k = max(0, len(new) - f)
        if k > len(U):
            k, new = len(U), new[: f + len(U)]
        best = 0
        for ev in itertools.combinations(U, k):
            nxt = frozenset((resd - set(ev)) | set(new))
            best = max(best, go(i + 1, nxt))
        return h + best

    return go(0, frozenset())


def test_hits_bounded_by_brute_force_opt():
    rng = np.random.default_rng(22)
    for trial in range(25):
        cap = int(rng.integers(2, 7))
        pool = [rng.integers(0, 1 << 17, 16 * int(rng.integers(1, 3))).astype(np.uint32)
                for _ in range(4)]
        reqs = []
        for _ in range(int(rng.integers(3, 11))):
            toks = np.concatenate([pool[i] for i in rng.integers(0, 4, rng.integers(1, 3))])
            reqs.append(toks)
        chains = tuple(tuple(chain_ref(t)) for t in reqs)
        opt = _opt_hits(cap, chains)
        for flags, types in ((1 | 4, 1), (0, 0), (2 | 1, 3)):
            R = replica(cap, K=3)
            L = LRU(cap)
            tot = lru = 0
            for i, t in enumerate(reqs):
                rc, res, *_ = R.admit_req(float(i + 1), t, np.full(len(t), types, np.uint8), [],
                                          flags, 1)
                tot += int(res[0])
                lru += L.admit(float(i + 1), list(chains[i]))[0]
            assert tot <= opt
            assert lru <= opt


def test_trace_invariants_capacity_partition_stage_order():
    tr = T.make("c1")
    cfg = C.policy_config(64, K=8)
    R = oracle.Replica(cfg)
    B = 16
    for i in range(tr["n"]):
        before = R.resident()
        by_hash = {int(h): (int(q), int(nt), int(bid)) for h, q, nt, bid in
                   zip(before["hash"], before["q"], before["ntok"], before["id"])}
        po, pl = int(tr["prompt_off"][i]), int(tr["prompt_len"][i])
        do, dl = int(tr["decode_off"][i]), int(tr["decode_len"][i])
        rc, res, vic, H, tau = R.admit_req(tr["arrival"][i], tr["tokens"][po:po + pl],
                                           tr["types"][po:po + pl], tr["tokens"][do:do + dl],
                                           tr["flags"][i], tr["spb"][i])
        assert rc == 0
        n = len(H)
        assert res[0] + res[1] == n
        assert n == -(-pl // B) + -(-dl // B)
        st = R.stats()
        assert st.resident <= 64
        assert sum(st.resident_by_queue) == st.resident
        # every hit's ancestors are resident (strict prefix)
        for j in range(int(res[0])):
            assert int(H[j]) in by_hash
        # stage order (Alg.1): EF victims first, ordered by (ntok, id)
        pin = {int(h) for h in H if int(h) in by_hash}
        ef = sorted((nt, bid) for hsh, (q, nt, bid) in by_hash.items()
                    if q == 0 and hsh not in pin)
        k = len(vic)
        e = min(k, len(ef))
        assert [int(v) for v in vic[:e]] == [bid for _, bid in ef[:e]]
        id2q = {bid: q for hsh, (q, nt, bid) in by_hash.items()}
        for v in vic[e:]:
            assert id2q[int(v)] != 0
        # victims were unpinned residents
        for v in vic:
            assert int(v) in id2q
            assert int(v) not in {by_hash[h][2] for h in pin}


def test_hand_traced_eviction_order():
    """Hand trace (C=4): two EF blocks (partial first), then scored queue by P."""
    R = replica(4, learn_flags=0, w=[1.0] * 5, alpha=[1.0] * 3)
    rng = np.random.default_rng(5)
    a = rng.integers(0, 1 << 17, 40).astype(np.uint32)   # 3 blocks: 16,16,8 tokens
    # request 1 at t=1: untemplated single-turn user blocks -> EF (ntok 16,16,8)
    rc, res, vic, H1, _ = R.admit_req(1.0, a, np.ones(40, np.uint8), [], 0, 0)
    assert list(vic) == []
    # request 2 at t=2: 1 system-prompt block -> STRUCT (o_b = 0 -> p = 1)
    b = rng.integers(0, 1 << 17, 16).astype(np.uint32)
    rc, res, vic, H2, _ = R.admit_req(2.0, b, np.zeros(16, np.uint8), [], 0, 1)
    assert list(vic) == []
    # request 3 at t=3: 3 new blocks -> evict 3: EF by (ntok, id): id2 (8 tok), id0, id1
    c = rng.integers(0, 1 << 17, 48).astype(np.uint32)
    rc, res, vic, H3, _ = R.admit_req(3.0, c, np.ones(48, np.uint8), [], 1 | 4, 0)
    assert list(vic) == [2, 0, 1]
    # request 4 at t=10: 2 new chat blocks -> evict 2 among STRUCT id3 (P=1/8) and chat
    # ids 4,5,6 (P = S(7; 4.15, 0.97)/7): S(7) ~ 0.9978 -> P ~ 0.1425 > 0.125
    d = rng.integers(0, 1 << 17, 32).astype(np.uint32)
    rc, res, vic, H4, _ = R.admit_req(10.0, d, np.ones(32, np.uint8), [], 1 | 4, 0)
    s7 = oracle.survival(7.0, 4.15, 0.97)
    assert s7 / 7.0 > 1.0 / 8.0
    assert list(vic) == [3, 4]


def test_errors_time_and_empty():
    R = replica(8)
    t = np.arange(16, dtype=np.uint32)
    rc, *_ = R.admit_req(5.0, t, np.ones(16, np.uint8), [], 0, 0)
    assert rc == 0
    rc, *_ = R.admit_req(4.0, t, np.ones(16, np.uint8), [], 0, 0)
    assert rc == -5  # SAE_E_TIME
    rc, v = R.evict(5, 6.0)
    assert rc == -3 and len(v) == 1  # SAE_E_EMPTY after evicting the one block
    rc, *_ = R.admit_req(7.0, np.zeros(0, np.uint32), np.zeros(0, np.uint8), [], 0, 0)
    assert rc == -1  # SAE_E_INVAL (L >= 1)
