"""Pins of the oracle's baseline / ablation modes (include/sae.h
SAE_MODE_*): LRU, LFU and Token-Weight-Only against textbook
reference policies written here from their definitions, with the replay's admission
semantics (pinning of the request's resident blocks, orphan refresh, overflow cap); and the
TTFT model prefill = L (1 - hit) on a hand case."""
import numpy as np
import pytest

import xxhash

import oracle
from paper_2605_18825_b200 import configs as C
from tests.test_oracle_hash import chain_ref


class RefPolicy:
    """Textbook LRU / LFU / w_tau/dt over one pool; blocks = {hash: [last, id, acc, tau]}."""

    def __init__(self, cap, mode, w=None, eps=1e-3):
        self.cap, self.mode, self.res, self.next_id = cap, mode, {}, 0
        self.w, self.eps = w, eps

    def key(self, b, now):
        last, bid, acc, tau = b
        if self.mode == C.MODE_LRU:
            return (last, last, bid)
        if self.mode == C.MODE_LFU:
            return (float(acc), last, bid)
        dt = now - last
        if dt < self.eps:
            dt = self.eps
        return (self.w[min(tau, 4)] / dt, last, bid)

    def admit(self, now, chain, taus):
        h = 0
        while h < len(chain) and chain[h] in self.res:
            h += 1
        pin = {x for x in chain if x in self.res}
        for j, x in enumerate(chain):
            if x in self.res:
                b = self.res[x]
                b[0] = now          # touch (hit or orphan)
                b[3] = taus[j]      # the block's type is overwritten (last writer)
                if j < h:
                    b[2] += 1       # an access only on a hit
        new = [j for j in range(h, len(chain)) if chain[j] not in self.res]
        f = self.cap - len(self.res)
        U = len(self.res) - len(pin)
        k = max(0, len(new) - f)
        if k > U:
            k, new = U, new[: f + U]
        cand = sorted((self.key(b, now), x) for x, b in self.res.items() if x not in pin)
        victims = []
        for _, x in cand[:k]:
            victims.append(self.res[x][1])
            del self.res[x]
        for j in new:
            self.res[chain[j]] = [now, self.next_id, 1, taus[j]]
            self.next_id += 1
        return h, victims


@pytest.mark.parametrize("mode", [C.MODE_LRU, C.MODE_LFU, C.MODE_TWO])
def test_baseline_modes_match_textbook_policies(mode):
    rng = np.random.default_rng(40 + mode)
    w = [2.0, 1.5, 1.0, 0.7, 0.1]
    for trial in range(4):
        cap = int(rng.integers(8, 40))
        p = dict(C.DEFAULT_PARAMS)
        p.update(mode=mode, w=w, learn_flags=0)
        R = oracle.Replica(C.policy_config(cap, params=p))
        ref = RefPolicy(cap, mode, w=w)
        pool = [rng.integers(0, 1 << 17, 16 * int(rng.integers(1, 5))).astype(np.uint32) for _ in range(12)]
        now = 0.0
        for step in range(200):
            toks = np.concatenate([pool[i] for i in rng.integers(0, 12, rng.integers(1, 4))])
            toks = toks[: len(toks) - int(rng.integers(0, 12))]
            types = rng.integers(0, 5, len(toks)).astype(np.uint8)
            dec = rng.integers(0, 1 << 17, int(rng.integers(0, 33))).astype(np.uint32)
            now += float(rng.choice([0.0, 1e-4, 0.7, 5.0, 60.0]))
            flags = int(rng.choice([0, 1, 3, 5]))
            rc, res, vic, H, tau = R.admit_req(now, toks, types, dec, flags, int(rng.integers(0, 3)))
            assert rc == 0
            chain = chain_ref(toks)
            # decode blocks chain from the last prompt block and start a new block (A34)
            prev = chain[-1]
            for s in range(0, len(dec), 16):
                blk = dec[s:s + 16].astype("<u4").tobytes()
                prev = xxhash.xxh64(int(prev).to_bytes(8, "little") + blk, seed=0).intdigest()
                chain.append(prev)
            assert [int(x) for x in H] == chain
            h, lv = ref.admit(now, chain, [int(t) for t in tau])
            assert res[0] == h, (mode, trial, step)
            assert [int(v) for v in vic] == lv, (mode, trial, step, list(vic), lv)
            st = R.stats()
            assert st.resident_by_queue[1] == st.resident     # one queue in the baselines


def test_fixed_param_mq_is_sae_with_learners_off():
    """Fixed-Param MQ = the multi-queue policy with learners off and the chat-fitted
    (mu, sigma) = (4.15, 0.97) for both multi-turn queues: no parameter ever moves."""
    from paper_2605_18825_b200 import tracegen as T
    tr = T.make("c1")
    p = dict(C.DEFAULT_PARAMS)
    p.update(learn_flags=0, mu=[4.15, 4.15], sigma=[0.97, 0.97])
    R = oracle.Replica(C.policy_config(64, K=8, params=p))
    res = R.replay(tr)
    assert res.stats.learner_firings > 10
    assert all(list(t.mu) == [4.15, 4.15] and list(t.w) == p["w"] for t in res.traj)


def test_ttft_prefill_model_hand_case():
    """prefill_tokens = prompt_length x (1 - hit_ratio): a 40-token prompt whose
    first 2 blocks (32 tokens) hit needs 8 prefill tokens."""
    from paper_2605_18825_b200 import ablation as A
    assert A.prefill_tokens(np.array([40, 16, 7]), np.array([32, 16, 0])).tolist() == [8, 0, 7]
