"""-m gpu parity: the CUDA path (through the C ABI) vs the CPU oracle on the same
seeded inputs, element by element: block hashes and types, per-request hit/miss/
matched/victim counts, the victim-id sequence, every learner snapshot, final
counters and parameters -- all bit-exact (SURVEY c.4: exactly one correct output)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2605_18825_b200 import configs as C
from paper_2605_18825_b200 import sae as S
from paper_2605_18825_b200 import tracegen as T
from tests.gpu_helpers import (assert_params_equal, assert_stats_equal, assert_traj_equal,
                               compare_replay, gpu_replay, u32, unpack)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c1():
    return T.make("c1")


@pytest.mark.parametrize("K", [8, 100])
def test_c1_replay_bit_exact(c1, K):
    compare_replay(c1, C.policy_config(64, K=K))


@pytest.mark.parametrize("flags", [0, C.L_TOKENS, C.L_DEFAULT | C.L_TOKEN_MULT,
                                   C.L_DEFAULT | C.L_QUEUE_RELATIVE, C.L_DEFAULT | C.L_ADAPTIVE_BETA])
def test_c1_learner_variants(c1, flags):
    p = dict(C.DEFAULT_PARAMS)
    p["learn_flags"] = flags
    compare_replay(c1, C.policy_config(64, K=8, params=p))


def test_c1_small_ghost_and_tiny_capacity(c1):
    compare_replay(c1, C.policy_config(16, K=5, ghost_capacity=7))


def test_mix_traces_several_tiles_and_ragged():
    # balanced and single-turn-dominant mixes, C spanning several 512-thread tiles
    for mix, cap in ((C.MIX_BAL, 700), (C.MIX_ST, 1500), (C.MIX_MT, 2304)):
        cfg = C.get("c2", n_requests=1500, mix=mix, seed=0x5AEC0100 + cap)
        tr = T.generate(cfg)
        T.materialize(tr)
        compare_replay(tr, C.policy_config(cap, K=100))


def test_c2_prefix_bit_exact():
    tr = T.make("c2", n_requests=6000)
    compare_replay(tr, C.policy_config(2304, K=100))


def test_lookup_matches_oracle(c1):
    pol = C.policy_config(64, K=8)
    cache, b, out = gpu_replay(c1, pol, lo=0, hi=120)
    R = oracle.Replica(pol)
    R.replay(c1, 0, 120)
    sub = T.single_batch(c1)
    hits = u32(cache.lookup(S.batch_to_torch(sub)))
    for i in range(c1["n"]):
        po, pl = int(c1["prompt_off"][i]), int(c1["prompt_len"][i])
        do, dl = int(c1["decode_off"][i]), int(c1["decode_len"][i])
        assert hits[i] == R.lookup(c1["tokens"][po:po + pl], c1["types"][po:po + pl],
                                   c1["tokens"][do:do + dl])
    # lookup changes nothing
    st = cache.stats(0)
    assert st.requests == 120


def test_evict_and_update_match_oracle(c1):
    pol = C.policy_config(64, K=8)
    cache, b, out = gpu_replay(c1, pol, lo=0, hi=100)
    R = oracle.Replica(pol)
    R.replay(c1, 0, 100)
    now = float(c1["arrival"][99]) + 1.0
    for k in (3, 10, 1):
        ids, n = cache.evict(0, k, now)
        rc, ref = R.evict(k, now)
        assert rc == 0
        assert int(n.item()) == len(ref)
        assert list(u32(ids)[:len(ref)]) == list(ref)
        now += 2.5
    cache.update(0)
    R.update()
    st = cache.stats(0)
    assert_params_equal(S.params_dict(st.params), R.params())
    assert_stats_equal(st, R.stats())
    assert_traj_equal(cache.traj(0), R.traj())


def test_evict_empty_raises_sticky(c1):
    pol = C.policy_config(64, K=8)
    cache, b, out = gpu_replay(c1, pol, lo=0, hi=10)
    live = cache.stats(0).resident
    ids, n = cache.evict(0, int(live) + 5, float(c1["arrival"][9]) + 1)
    with pytest.raises(S.SaeError) as e:
        cache.sync()
    assert e.value.status == -3
    assert int(n.item()) == live


def test_time_backwards_sticky(c1):
    pol = C.policy_config(64, K=8)
    cache, b, out = gpu_replay(c1, pol, lo=0, hi=20)
    bad = T.single_batch(c1)
    bad = {k: (v[:5] if hasattr(v, "__len__") and k not in ("tokens", "types") else v)
           for k, v in bad.items()}
    bad["n"] = 5
    cache.admit_batch(S.batch_to_torch(bad))
    with pytest.raises(S.SaeError) as e:
        cache.sync()
    assert e.value.status == -5


def test_multi_replica_parameter_points():
    """C5-shaped: several replicas (interleaved-free runs) with different parameter
    points, each equal to its own oracle replay."""
    cfg = C.get("c5", n_requests=800, capacity=256)
    traces = []
    for sd in range(2):
        t = T.generate(C.get("c5", n_requests=800), seed=0x5AEC1000 + sd)
        T.materialize(t)
        traces.append(t)
    R = 6
    rep_of = [r % 2 for r in range(R)]
    batch = T.replicate(traces, rep_of)
    pol = C.policy_config(256, K=50)
    cache = S.SaeCache(256, n_replicas=R, policy=pol, traj_capacity=1 << 14)
    points = [0, 7, 29, 30, 31, 12]
    for r in range(R):
        cache.set_params(r, C.c5_point_params(points[r]))
    b = S.batch_to_torch(batch)
    out = cache.admit_batch(b)
    torch.cuda.synchronize()
    o4, _ = unpack(out, batch["n"])
    vo = out["victim_off"].cpu().numpy()
    vids = u32(out["victim_ids"])
    off = 0
    for r in range(R):
        tr = traces[rep_of[r]]
        p = dict(pol)
        p["params"] = C.c5_point_params(points[r])
        O = oracle.Replica(p)
        ref = O.replay(tr)
        n = tr["n"]
        assert np.array_equal(o4[off:off + n], ref.out4), r
        got = np.concatenate([vids[vo[off + i]:vo[off + i] + o4[off + i, 3]] for i in range(n)])
        assert np.array_equal(got, ref.victims), r
        st = cache.stats(r)
        assert_stats_equal(st, ref.stats)
        assert_traj_equal(cache.traj(r), ref.traj)
        assert_params_equal(S.params_dict(st.params), O.params())
        off += n


@pytest.mark.parametrize("chunks", [2, 7])
def test_task_split_replay_matches_oracle(chunks, monkeypatch):
    """Task-split persistent replay (sae.cu d.nchunk, forced with SAE_CHUNKS): each replica's
    run is replayed as consecutive chunks taken from one task counter by whichever CTA is
    free, the state crossing SMs through release/acquire flags; uneven and empty chunks
    (runs shorter than the chunk count) included.  Every replica equals its oracle replay."""
    monkeypatch.setenv("SAE_CHUNKS", str(chunks))
    traces = []
    for sd in range(3):
        t = T.generate(C.get("c5", n_requests=500), seed=0x5AEC2000 + sd)
        T.materialize(t)
        traces.append(t)
    R = 9
    rep_of = [r % 3 for r in range(R)]
    pol = C.policy_config(256, K=40)
    cache = S.SaeCache(256, n_replicas=R, policy=pol, traj_capacity=1 << 14)
    assert cache.layout()["chunks"] == chunks
    for r in range(R):
        cache.set_params(r, C.c5_point_params((5 * r) % 32))
    # three launches per replica run: 3 requests (fewer than 7 chunks), then the rest in two
    cuts = [0, 3, 200, 500]
    got = {r: ([], []) for r in range(R)}
    for a, z in zip(cuts[:-1], cuts[1:]):
        part = [{**{k: t[k][a:z] for k in ("arrival", "prompt_off", "prompt_len", "decode_off",
                                            "decode_len", "flags", "spb")},
                 "n": z - a, "tokens": t["tokens"], "types": t["types"], "n_tokens": t["n_tokens"]}
                for t in traces]
        batch = T.replicate(part, rep_of)
        out = cache.admit_batch(S.batch_to_torch(batch))
        torch.cuda.synchronize()
        o4, _ = unpack(out, batch["n"])
        vo = out["victim_off"].cpu().numpy()
        vids = u32(out["victim_ids"])
        for r in range(R):
            off = r * (z - a)
            got[r][0].append(o4[off:off + z - a])
            got[r][1].extend(int(v) for i in range(z - a) for v in vids[vo[off + i]:vo[off + i] + o4[off + i, 3]])
    for r in range(R):
        p = dict(pol)
        p["params"] = C.c5_point_params((5 * r) % 32)
        O = oracle.Replica(p)
        ref = O.replay(traces[rep_of[r]])
        assert np.array_equal(np.concatenate(got[r][0]), ref.out4), r
        assert got[r][1] == [int(v) for v in ref.victims], r
        assert_stats_equal(cache.stats(r), ref.stats)
        assert_traj_equal(cache.traj(r), ref.traj)


def test_gen_tokens_matches_numpy():
    tr = T.generate(C.get("c2", n_requests=500))
    T.materialize(tr)
    allp, dst = T.piece_table(tr)
    tok, ty = S.gen_tokens(tr["tseed"], allp, dst, tr["n_tokens"])
    assert np.array_equal(u32(tok)[:tr["n_tokens"]], tr["tokens"])
    assert np.array_equal(ty.cpu().numpy()[:tr["n_tokens"]], tr["types"])


def test_c5_mean_w_sync_matches_oracle():
    """mean_w@E sync: after every epoch of E requests per replica the token
    weights of each parameter point become the fixed-order mean over its seeds."""
    from paper_2605_18825_b200 import replicas as RP
    npts, nseeds, E, epochs = 32, 2, 150, 3
    R = npts * nseeds
    traces = []
    for sd in range(nseeds):
        t = T.generate(C.get("c5", n_requests=E * epochs), seed=0x5AEC1000 + sd)
        T.materialize(t)
        traces.append(t)
    pol = C.policy_config(256, K=40)
    cache = S.SaeCache(256, n_replicas=R, policy=pol, traj_capacity=1 << 12)
    refs = []
    for r in range(R):
        sd, pt = RP.layout(r, npts)
        cache.set_params(r, C.c5_point_params(pt))
        p = dict(pol)
        p["params"] = C.c5_point_params(pt)
        refs.append(oracle.Replica(p))
    offs = np.cumsum([0] + [t["n_tokens"] for t in traces])
    tok = np.concatenate([t["tokens"] for t in traces])
    typ = np.concatenate([t["types"] for t in traces])
    for ep in range(epochs):
        lo, hi = ep * E, (ep + 1) * E
        cols = {k: [] for k in ("arrival", "prompt_off", "prompt_len", "decode_off", "decode_len",
                                "flags", "spb", "replica")}
        for r in range(R):
            t = traces[RP.layout(r, npts)[0]]
            for k in ("arrival", "prompt_len", "decode_len", "flags", "spb"):
                cols[k].append(t[k][lo:hi])
            o = np.uint64(offs[RP.layout(r, npts)[0]])
            cols["prompt_off"].append(t["prompt_off"][lo:hi] + o)
            cols["decode_off"].append(t["decode_off"][lo:hi] + o)
            cols["replica"].append(np.full(hi - lo, r, np.uint32))
        bb = {k: np.concatenate(v) for k, v in cols.items()}
        bb["n"], bb["tokens"], bb["types"] = len(bb["arrival"]), tok, typ
        out = cache.admit_batch(S.batch_to_torch(bb))
        RP.sync_mean_w(cache, npts)
        torch.cuda.synchronize()
        o4, _ = unpack(out, bb["n"])
        for r in range(R):
            t = traces[RP.layout(r, npts)[0]]
            res = refs[r].replay(t, lo, hi, want_hashes=False)
            assert np.array_equal(o4[r * E:(r + 1) * E], res.out4), (ep, r)
        newp = oracle.point_mean_w([x.params() for x in refs], npts)
        for r in range(R):
            refs[r].set_params(newp[r])
    for r in range(R):
        assert_params_equal(S.params_dict(cache.stats(r).params), refs[r].params())


def test_c2_prefix_adaptive_beta():
    """The adaptive EMA factor of LognormalParams (A28) over a C2 prefix."""
    p = dict(C.DEFAULT_PARAMS)
    p["learn_flags"] = C.L_DEFAULT | C.L_ADAPTIVE_BETA
    compare_replay(T.make("c2", n_requests=6000), C.policy_config(2304, params=p))


def test_admit_batch_host_pipelined_matches_oracle():
    """The end-to-end call sae_admit_batch_host (host buffers, inputs staged in two slots on
    the library's copy stream, the next call's copies overlapping the current replay), issued
    back to back with two calls in flight exactly as bench.py's e2e loop does, reading each
    call's pinned outputs only after the next call is queued: per-request outputs and the
    victim-id sequence equal the oracle's replay of the same trace."""
    tr = T.make("c2", n_requests=3000)
    pol = C.policy_config(2304, K=100)
    cache = S.SaeCache(2304, policy=pol)
    tok_h = torch.from_numpy(tr["tokens"].view(np.int32)).pin_memory()
    typ_h = torch.from_numpy(tr["types"]).pin_memory()
    tok_d = torch.zeros(tr["n_tokens"], dtype=torch.int32, device="cuda")
    typ_d = torch.zeros(tr["n_tokens"], dtype=torch.uint8, device="cuda")
    cuts = [0, 1, 400, 401, 1200, 2000, 3000]        # incl. one-request batches
    pend, got4, gotv = [], [], []

    def take(res, n):
        o4 = np.stack([res[k].numpy()[:n].view(np.uint32) for k in
                       ("hit_blocks", "miss_blocks", "matched_tokens", "n_victims")], 1)
        vo = res["victim_off"].numpy()
        vids = res["victim_ids"].numpy().view(np.uint32)
        got4.append(o4.copy())
        gotv.extend(int(v) for i in range(n) for v in vids[vo[i] - vo[0]:vo[i] - vo[0] + o4[i, 3]])

    for a, z in zip(cuts[:-1], cuts[1:]):
        hb = {k: tr[k][a:z] for k in ("arrival", "prompt_off", "prompt_len", "decode_off",
                                       "decode_len", "flags", "spb")}
        hb.update(n=z - a, replica=np.zeros(z - a, np.uint32), tokens=np.zeros(1, np.uint32),
                  types=np.zeros(1, np.uint8))
        hp = S.batch_to_torch(hb, pin=True)
        lo = int(hb["prompt_off"].min())
        hi = int((hb["decode_off"] + hb["decode_len"].astype(np.uint64)).max())
        res, _, _ = cache.admit_batch_host(hp, tok_h, typ_h, tok_d, typ_d, lo, hi)
        ev = torch.cuda.Event()
        ev.record()
        pend.append((ev, res, z - a))
        if len(pend) > 1:
            evp, rp, n = pend.pop(0)
            evp.synchronize()
            take(rp, n)
    torch.cuda.synchronize()
    for evp, rp, n in pend:
        take(rp, n)
    ref = oracle.Replica(pol).replay(tr, 0, 3000)
    assert np.array_equal(np.concatenate(got4), ref.out4)
    assert gotv == [int(v) for v in ref.victims]
