"""Hashing / prefix-lookup pins (SURVEY c.7): official XXH64 vectors, the python
``xxhash`` package as an independent implementation of the chained byte layout,
SPEC S:53-55 / S:62-64 hand cases and the median-token rule."""
import numpy as np
import xxhash

import oracle
from paper_2605_18825_b200 import configs as C

SEED = C.HASH_SEED


def test_xxh64_official_vectors():
    assert oracle.xxh64(b"") == 0xEF46DB3751D8E999
    assert oracle.xxh64(b"a") == 0xD24EC4F1A98C6E5B
    assert oracle.xxh64(b"abc") == 0x44BC2CF5AD770999


def test_xxh64_matches_python_xxhash_all_lengths():
    rng = np.random.default_rng(7)
    for n in range(0, 200):
        b = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        for seed in (0, 1, 0xFFFFFFFFFFFFFFFF):
            assert oracle.xxh64(b, seed) == xxhash.xxh64(b, seed=seed).intdigest()


def chain_ref(tokens, B=16, seed=SEED):
    """Chained block hash via the python xxhash package (independent)."""
    out = []
    prev = seed
    for s in range(0, len(tokens), B):
        blk = np.asarray(tokens[s:s + B], np.uint32)
        data = int(prev).to_bytes(8, "little") + blk.astype("<u4").tobytes()
        prev = xxhash.xxh64(data, seed=0).intdigest()
        out.append(prev)
    return out


def test_block_hash_chain_layout():
    rng = np.random.default_rng(8)
    toks = rng.integers(0, 1 << 17, 16 * 5 + 7).astype(np.uint32)
    ref = chain_ref(toks)
    prev = SEED
    for j, s in enumerate(range(0, len(toks), 16)):
        prev = oracle.block_hash(prev, toks[s:s + 16])
        assert prev == ref[j]


def _replica(cap=64, K=100, **pover):
    p = dict(C.DEFAULT_PARAMS)
    p.update(pover)
    return oracle.Replica(C.policy_config(cap, K=K, params=p))


def test_chain_hashes_from_replay_match_python_xxhash():
    rng = np.random.default_rng(9)
    R = _replica()
    toks = rng.integers(0, 1 << 17, 53).astype(np.uint32)
    types = np.zeros(53, np.uint8)
    dec = rng.integers(0, 1 << 17, 20).astype(np.uint32)
    rc, res, vic, H, tau = R.admit_req(1.0, toks, types, dec, 0, 2)
    assert rc == 0
    ref = chain_ref(toks)
    # decode blocks start a new block chained from the last prompt block (A34)
    prev = ref[-1]
    for s in range(0, 20, 16):
        data = int(prev).to_bytes(8, "little") + dec[s:s + 16].astype("<u4").tobytes()
        prev = xxhash.xxh64(data).intdigest()
        ref.append(prev)
    assert list(H) == ref
    assert list(tau) == [0, 0, 0, 0, 5, 5]


def test_prefix_hits_spec_examples():
    # exact repeat -> all hits; 32 shared tokens -> 2 hits; 40 cold tokens -> 3 misses
    rng = np.random.default_rng(10)
    R = _replica(cap=1000)
    A = rng.integers(0, 1 << 17, 64).astype(np.uint32)
    ty = np.ones(64, np.uint8)
    rc, res, *_ = R.admit_req(1.0, A, ty, [], 0, 0)
    assert rc == 0 and res[0] == 0 and res[1] == 4
    rc, res, *_ = R.admit_req(2.0, A, ty, [], 0, 0)
    assert res[0] == 4 and res[1] == 0 and res[2] == 64
    Bt = A.copy()
    Bt[32:] = rng.integers(0, 1 << 17, 32)
    rc, res, *_ = R.admit_req(3.0, Bt, ty, [], 0, 0)
    assert res[0] == 2 and res[2] == 32
    cold = rng.integers(0, 1 << 17, 40).astype(np.uint32)
    rc, res, *_ = R.admit_req(4.0, cold, ty[:40], [], 0, 0)
    assert res[0] == 0 and res[1] == 3


def test_median_token_type_rule():
    # P:320 "type of the median token"; A3: index floor(n/2)
    R = _replica()
    toks = np.arange(16 * 2 + 3, dtype=np.uint32)
    ty = np.zeros(35, np.uint8)
    ty[10:16] = 1            # block 0: 10 sys + 6 user -> index 8 -> sys
    ty[16:23] = 0            # block 1: 7 sys + 9 user -> index 8 -> user
    ty[23:32] = 1
    ty[32:35] = [3, 2, 3]    # partial 3-token block -> index 1 -> tool
    rc, res, vic, H, tau = R.admit_req(1.0, toks, ty, [], 0, 0)
    assert list(tau) == [0, 1, 2]


def test_prefix_match_maximality_brute_force():
    """Hit count = longest chained prefix resident (brute force over <= 64 blocks)."""
    rng = np.random.default_rng(11)
    for trial in range(30):
        R = _replica(cap=64)
        pool = [rng.integers(0, 50, 16 * rng.integers(1, 5)).astype(np.uint32) for _ in range(6)]
        now = 0.0
        for step in range(12):
            # requests are concatenations of pool segments (lots of shared prefixes)
            segs = [pool[i] for i in rng.integers(0, 6, rng.integers(1, 4))]
            toks = np.concatenate(segs)
            ty = np.ones(len(toks), np.uint8)
            before = set(int(x) for x in R.resident()["hash"])
            chain = chain_ref(toks)
            brute = 0
            while brute < len(chain) and chain[brute] in before:
                brute += 1
            assert R.lookup(toks, ty, []) == brute
            now += 1.0
            rc, res, *_ = R.admit_req(now, toks, ty, [], 1, 0)
            assert rc == 0 and res[0] == brute
            assert res[0] + res[1] == len(chain)
            assert R.stats().resident <= 64
