"""Seeded synthetic trace generator (the shared INPUT of the GPU path and the oracle).

Holds none of the method's arithmetic: it only draws requests shaped like the
paper's synthetic workloads (Appendix D; Table 2 mixes P:884-888;
log-normal inter-turn gaps P:185; turn counts P:1109-1110; the
session predictor's confusion matrix P:1179 for turn-0 ``is_multi_turn``) and
materialises token ids with a counter-based SplitMix64:

    tok(stream, pos) = SM(SM(seed ^ SM(stream)) ^ pos) mod 2**17

Template tokens are keyed by (category, template id) so they repeat across
requests; content tokens are keyed by (session, turn, part) so they are unique
("cross-session reuse < 0.01%").  The recipe and every chosen length
are stated in DESIGN.md §Inputs.

Output: a dict of numpy arrays in the ``sae_batch`` layout (include/sae.h):
``arrival f64, prompt_off u64, prompt_len u32, decode_off u64, decode_len u32,
flags u8, spb u32, tokens u32, types u8`` plus piece tables so tokens can be
(re)materialised for any subset of requests (numpy here, or the CUDA
``sae_gen_tokens`` on the device).
"""
from __future__ import annotations

import numpy as np

from . import configs as C

M64 = (1 << 64) - 1
_G = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

CATS = ["chat", "agent", "tool_use", "programming", "doc_qa"]

# Per-category recipe (SURVEY §8(d) "Trace generator"; medians in tokens, log-normal
# with sigma_len = 0.6; template lengths fixed per template id).
CAT_SPEC = {
    "chat": dict(n_tpl=16, tpl_len=64, tpl_med=None, sys_frac=1.0, in0=(C.USER, 100),
                 inN=(C.USER, 100), extra=None, out=200, cot=0.3, turns=3.6,
                 gap=(4.82, 1.25), zipf=None),
    "agent": dict(n_tpl=64, tpl_len=384, tpl_med=None, sys_frac=1.0 / 3.0, in0=(C.USER, 100),
                  inN=(C.TOOL, 250), extra=None, out=200, cot=0.3, turns=6.0,
                  gap=(2.28, 1.34), zipf=None),
    "tool_use": dict(n_tpl=1 << 10, tpl_len=None, tpl_med=510, sys_frac=0.3, in0=(C.USER, 90),
                     inN=None, extra=None, out=80, cot=0.0, turns=1.0, gap=None, zipf=0.8),
    "programming": dict(n_tpl=1 << 8, tpl_len=None, tpl_med=200, sys_frac=1.0, in0=(C.USER, 300),
                        inN=None, extra=None, out=300, cot=0.3, turns=1.0, gap=None, zipf=0.8),
    "doc_qa": dict(n_tpl=16, tpl_len=None, tpl_med=80, sys_frac=1.0, in0=(C.USER, 700),
                   inN=None, extra=(C.USER, 30), out=100, cot=0.0, turns=1.0, gap=None, zipf=None),
}
SIGMA_LEN = 0.6
CARRY_COT_P = 0.1
REQ_INTERVAL = 0.03          # mean request inter-arrival (mid of P:410's sweep)
P_PRED_CONT = 175.0 / 190.0  # P(pred multi-turn | continues)
P_PRED_SINGLE = 71.0 / 186.0  # P(pred multi-turn | single)


# ---------------------------------------------------------------------------
# counter-based token PRNG
# ---------------------------------------------------------------------------
def splitmix(x: np.ndarray) -> np.ndarray:
    z = x.astype(np.uint64) + _G
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def splitmix_int(x: int) -> int:
    z = (x + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def stream_key(tseed: int, stream: np.ndarray) -> np.ndarray:
    """Per-piece key SM(seed ^ SM(stream))."""
    return splitmix(np.uint64(tseed) ^ splitmix(stream))


def tokens_of(key: np.ndarray, pos: np.ndarray) -> np.ndarray:
    return (splitmix(key ^ pos.astype(np.uint64)) & np.uint64(0x1FFFF)).astype(np.uint32)


def tpl_stream(cat: int, tid) -> np.ndarray:
    return (np.uint64(1) << np.uint64(60)) | (np.uint64(cat) << np.uint64(32)) | np.asarray(tid, np.uint64)


def content_stream(session, turn, part) -> np.ndarray:
    s = np.asarray(session, np.uint64)
    t = np.asarray(turn, np.uint64)
    p = np.asarray(part, np.uint64)
    return (np.uint64(2) << np.uint64(60)) | (s << np.uint64(12)) | (t << np.uint64(2)) | p


# ---------------------------------------------------------------------------
def _lognorm_len(rng, med, n, scale):
    m = max(1.0, med * scale)
    x = np.exp(rng.normal(np.log(m), SIGMA_LEN, n))
    return np.clip(np.rint(x), 1, max(2, 20 * m)).astype(np.int64)


def _zipf_sample(rng, n_items, a, n):
    w = np.arange(1, n_items + 1, dtype=np.float64) ** (-a)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    idx = np.searchsorted(cdf, rng.random(n), side="right")
    # random permutation of ranks -> template ids (popularity not tied to id order)
    perm = rng.permutation(n_items)
    return perm[np.minimum(idx, n_items - 1)]


def _sessions(cfg, rng, ws):
    """Session metadata: category, turns, start time, per-turn arrival times."""
    n = cfg["n_requests"]
    mean_turns = np.array([CAT_SPEC[c]["turns"] for c in CATS])
    Et = float((ws * mean_turns).sum())
    S = int(np.ceil(n * 1.6 / Et)) + 64
    cat = rng.choice(5, S, p=ws)
    turns = np.ones(S, np.int64)
    for ci, c in enumerate(CATS):
        if CAT_SPEC[c]["turns"] > 1.0:
            m = cat == ci
            turns[m] = rng.geometric(1.0 / CAT_SPEC[c]["turns"], int(m.sum()))
    turns = np.minimum(turns, 200)
    starts = np.cumsum(rng.exponential(Et * REQ_INTERVAL, S))
    T = int(turns.sum())
    sess = np.repeat(np.arange(S), turns)
    first = np.zeros(S + 1, np.int64)
    first[1:] = np.cumsum(turns)
    tidx = np.arange(T) - first[sess]
    gaps = np.zeros(T)
    for ci, c in enumerate(CATS):
        g = CAT_SPEC[c]["gap"]
        if g is None:
            continue
        m = (cat[sess] == ci) & (tidx > 0)
        gaps[m] = np.exp(rng.normal(g[0], g[1], int(m.sum())))
    cg = np.cumsum(gaps)
    base = cg[first[:-1]]
    t = starts[sess] + (cg - base[sess])
    return cat, turns, sess, tidx, t


def generate(cfg: dict, seed: int | None = None) -> dict:
    """Generate one single-replica trace for config ``cfg`` (configs.CONFIGS entry)."""
    seed = cfg["seed"] if seed is None else seed
    n = int(cfg["n_requests"])
    scale = float(cfg.get("len_scale", 1.0))
    mix = np.asarray(cfg["mix"], np.float64)
    mean_turns = np.array([CAT_SPEC[c]["turns"] for c in CATS])
    ws = mix / mean_turns
    ws /= ws.sum()
    # calibration rounds so that REQUEST shares match Table 2 after edge truncation
    for _ in range(12):
        rng = np.random.default_rng([seed & M64, 1])
        cat, turns, sess, tidx, t = _sessions(cfg, rng, ws)
        us = np.rint(t * 1e6).astype(np.int64)
        order = np.lexsort((tidx, sess, us))[:n]
        got = np.bincount(cat[sess[order]], minlength=5) / n
        adj = np.where(got > 0, mix / np.maximum(got, 1e-12), 1.0)
        if np.all(np.abs(got - mix) < 0.01):
            break
        ws = ws * adj
        ws /= ws.sum()
    rng2 = np.random.default_rng([seed & M64, 2])
    S = len(turns)
    # continuation flag and turn-0 prediction (A33)
    cont = turns > 1
    pred = np.where(cont, rng2.random(S) < P_PRED_CONT, rng2.random(S) < P_PRED_SINGLE)
    # templates per session
    tpl_id = np.zeros(S, np.int64)
    tpl_len_of = {}
    for ci, c in enumerate(CATS):
        spec = CAT_SPEC[c]
        ntpl, tlen = spec["n_tpl"], spec["tpl_len"]
        ov = cfg.get("tpl_override", {}).get(c)
        if ov is not None:
            ntpl, tlen = ov
        ntpl = int(cfg.get("n_tpl", {}).get(c, ntpl))
        trng = np.random.default_rng([seed & M64, 100 + ci])
        if tlen is not None:
            L = np.full(ntpl, int(tlen) if ov is not None else max(1, int(round(tlen * scale))), np.int64)
        else:
            L = _lognorm_len(trng, spec["tpl_med"], ntpl, scale)
            L = np.maximum(L, 1)
        tpl_len_of[ci] = L
        m = cat == ci
        cnt = int(m.sum())
        if spec["zipf"] is not None:
            tpl_id[m] = _zipf_sample(trng, ntpl, spec["zipf"], cnt)
        else:
            tpl_id[m] = trng.integers(0, ntpl, cnt)
    # per-turn content lengths (drawn for every turn of every session)
    T = len(sess)
    in_len = np.zeros(T, np.int64)
    in_type = np.zeros(T, np.int64)
    ex_len = np.zeros(T, np.int64)
    out_len = np.zeros(T, np.int64)
    cot_len = np.zeros(T, np.int64)
    carry_cot = rng2.random(T) < CARRY_COT_P
    for ci, c in enumerate(CATS):
        spec = CAT_SPEC[c]
        m = cat[sess] == ci
        k = int(m.sum())
        if k == 0:
            continue
        m0 = m & (tidx == 0)
        mN = m & (tidx > 0)
        in_len[m0] = _lognorm_len(rng2, spec["in0"][1], int(m0.sum()), scale)
        in_type[m0] = spec["in0"][0]
        if spec["inN"] is not None and mN.any():
            in_len[mN] = _lognorm_len(rng2, spec["inN"][1], int(mN.sum()), scale)
            in_type[mN] = spec["inN"][0]
        if spec["extra"] is not None:
            ex_len[m] = _lognorm_len(rng2, spec["extra"][1], k, scale)
        out_len[m] = _lognorm_len(rng2, spec["out"], k, scale)
        cot_len[m] = np.rint(out_len[m] * spec["cot"]).astype(np.int64)
    first = np.zeros(S + 1, np.int64)
    first[1:] = np.cumsum(turns)

    # ---- pieces per selected request, in arrival order ------------------------------
    tseed = seed & M64
    p_stream, p_start, p_len, p_type = [], [], [], []
    req_pp = np.zeros(n + 1, np.int64)   # prompt piece ranges
    req_dp = np.zeros(n + 1, np.int64)   # decode piece ranges (separate table)
    d_stream, d_start, d_len, d_type = [], [], [], []
    flags = np.zeros(n, np.uint8)
    spb = np.zeros(n, np.uint32)
    req_cat = np.zeros(n, np.uint8)
    req_sess = np.zeros(n, np.int64)
    req_turn = np.zeros(n, np.int64)
    ag_bit = np.array([0, 2, 0, 0, 0], np.uint8)
    for i, r in enumerate(order):
        s = int(sess[r]); tt = int(tidx[r]); ci = int(cat[s]); spec = CAT_SPEC[CATS[ci]]
        req_cat[i], req_sess[i], req_turn[i] = ci, s, tt
        tl = int(tpl_len_of[ci][tpl_id[s]])
        nsys = int(round(tl * spec["sys_frac"]))
        ts = int(tpl_stream(ci, tpl_id[s]))
        if nsys > 0:
            p_stream.append(ts); p_start.append(0); p_len.append(nsys); p_type.append(C.SYS)
        if tl - nsys > 0:
            p_stream.append(ts); p_start.append(nsys); p_len.append(tl - nsys); p_type.append(C.TOOL)
        spb[i] = tl // 16
        base = first[s]
        for u in range(tt + 1):
            g = base + u
            p_stream.append(int(content_stream(s, u, 0))); p_start.append(0)
            p_len.append(int(in_len[g])); p_type.append(int(in_type[g]))
            if ex_len[g] > 0:
                p_stream.append(int(content_stream(s, u, 2))); p_start.append(0)
                p_len.append(int(ex_len[g])); p_type.append(C.USER)
            if u < tt:  # carried history of turn u
                os_ = int(content_stream(s, u, 1))
                cl, ol = int(cot_len[g]), int(out_len[g])
                if carry_cot[g] and cl > 0:
                    p_stream.append(os_); p_start.append(0); p_len.append(cl); p_type.append(C.COT)
                if ol - cl > 0:
                    p_stream.append(os_); p_start.append(cl); p_len.append(ol - cl); p_type.append(C.RESP)
        req_pp[i + 1] = len(p_stream)
        g = base + tt
        os_ = int(content_stream(s, tt, 1))
        cl, ol = int(cot_len[g]), int(out_len[g])
        if cl > 0:
            d_stream.append(os_); d_start.append(0); d_len.append(cl); d_type.append(C.COT)
        if ol - cl > 0:
            d_stream.append(os_); d_start.append(cl); d_len.append(ol - cl); d_type.append(C.RESP)
        req_dp[i + 1] = len(d_stream)
        mt = tt > 0 or bool(pred[s])
        flags[i] = (1 if mt else 0) | int(ag_bit[ci]) | (4 if tt > 0 else 0)

    P = dict(stream=np.array(p_stream, np.uint64), start=np.array(p_start, np.int64),
             len=np.array(p_len, np.int64), type=np.array(p_type, np.uint8))
    D = dict(stream=np.array(d_stream, np.uint64), start=np.array(d_start, np.int64),
             len=np.array(d_len, np.int64), type=np.array(d_type, np.uint8))
    plen = np.add.reduceat(P["len"], req_pp[:-1]) if n else np.zeros(0, np.int64)
    plen = np.where(np.diff(req_pp) > 0, plen, 0)
    dl = np.zeros(n, np.int64)
    nz = np.diff(req_dp) > 0
    if len(D["len"]):
        sums = np.add.reduceat(D["len"], np.minimum(req_dp[:-1], len(D["len"]) - 1))
        dl = np.where(nz, sums, 0)
    tot = plen + dl
    prompt_off = np.zeros(n, np.uint64)
    prompt_off[1:] = np.cumsum(tot)[:-1].astype(np.uint64)
    decode_off = prompt_off + plen.astype(np.uint64)
    us = np.rint(t[order] * 1e6).astype(np.int64)
    # strictly increasing, >= 1 us apart (tracegen invariant)
    us = np.maximum.accumulate(us - np.arange(n)) + np.arange(n)
    arrival = us.astype(np.float64) / 1e6
    tr = dict(n=n, seed=seed, tseed=tseed, arrival=arrival,
              prompt_off=prompt_off, prompt_len=plen.astype(np.uint32),
              decode_off=decode_off, decode_len=dl.astype(np.uint32),
              flags=flags, spb=spb, category=req_cat, session=req_sess, turn=req_turn,
              pieces=P, piece_off=req_pp, dpieces=D, dpiece_off=req_dp,
              n_tokens=int(tot.sum()), continues=cont[req_sess])
    return tr


def materialize(tr: dict, chunk: int = 1 << 23) -> dict:
    """Fill tr['tokens'] (u32) and tr['types'] (u8) for the whole arena (numpy)."""
    N = tr["n_tokens"]
    tokens = np.zeros(N, np.uint32)
    types = np.zeros(N, np.uint8)
    for pk, off_name, base_name in (("pieces", "piece_off", "prompt_off"),
                                     ("dpieces", "dpiece_off", "decode_off")):
        Pc = tr[pk]
        if len(Pc["len"]) == 0:
            continue
        po = tr[off_name]
        n = tr["n"]
        req_of_piece = np.repeat(np.arange(n), np.diff(po))
        # destination start of each piece inside the arena
        within = np.zeros(len(Pc["len"]), np.int64)
        cs = np.cumsum(Pc["len"])
        first_piece_cs = np.concatenate([[0], cs])[po[:-1]]
        within = np.concatenate([[0], cs[:-1]]) - first_piece_cs[req_of_piece]
        dst = tr[base_name][req_of_piece].astype(np.int64) + within
        keys = stream_key(tr["tseed"], Pc["stream"])
        # expand in chunks of pieces
        i = 0
        npcs = len(Pc["len"])
        while i < npcs:
            j = i
            acc = 0
            while j < npcs and acc < chunk:
                acc += int(Pc["len"][j]); j += 1
            L = Pc["len"][i:j]
            pid = np.repeat(np.arange(i, j), L)
            first_tok = np.concatenate([[0], np.cumsum(L)[:-1]])
            k = np.arange(len(pid)) - np.repeat(first_tok, L)
            pos = Pc["start"][pid] + k
            d = dst[pid] + k
            tokens[d] = tokens_of(keys[pid], pos)
            types[d] = Pc["type"][pid]
            i = j
    tr["tokens"] = tokens
    tr["types"] = types
    return tr


def piece_table(tr: dict):
    """The trace's token pieces (prompt then decode) and each piece's destination in the
    arena, in the layout materialize() fills -- the input of the device generator K7
    (sae_gen_tokens), which writes the same bytes on the GPU."""
    def dst_of(pk, off, base):
        po = tr[off]
        req = np.repeat(np.arange(tr["n"]), np.diff(po))
        cs = np.cumsum(tr[pk]["len"])
        first = np.concatenate([[0], cs])[po[:-1]]
        within = np.concatenate([[0], cs[:-1]]) - first[req]
        return tr[base][req].astype(np.int64) + within
    P, D = tr["pieces"], tr["dpieces"]
    allp = {k: np.concatenate([P[k], D[k]]) for k in ("stream", "start", "len", "type")}
    dst = np.concatenate([dst_of("pieces", "piece_off", "prompt_off"),
                          dst_of("dpieces", "dpiece_off", "decode_off")])
    return allp, dst


def make(name: str, materialize_tokens: bool = True, **over) -> dict:
    cfg = C.get(name, **over)
    tr = generate(cfg)
    tr["config"] = cfg
    if materialize_tokens:
        materialize(tr)
    return tr


def replicate(traces: list, replica_of: list) -> dict:
    """Batch of several replicas (grouped, arrival order within each) sharing one token
    arena: replica r uses trace replica_of[r]."""
    offs = np.zeros(len(traces) + 1, np.int64)
    for i, t in enumerate(traces):
        offs[i + 1] = offs[i] + t["n_tokens"]
    tokens = np.concatenate([t["tokens"] for t in traces])
    types = np.concatenate([t["types"] for t in traces])
    cols = {k: [] for k in ("arrival", "prompt_off", "prompt_len", "decode_off", "decode_len",
                            "flags", "spb", "replica")}
    for r, ti in enumerate(replica_of):
        t = traces[ti]
        cols["arrival"].append(t["arrival"])
        cols["prompt_off"].append(t["prompt_off"] + np.uint64(offs[ti]))
        cols["decode_off"].append(t["decode_off"] + np.uint64(offs[ti]))
        for k in ("prompt_len", "decode_len", "flags", "spb"):
            cols[k].append(t[k])
        cols["replica"].append(np.full(t["n"], r, np.uint32))
    out = {k: np.concatenate(v) for k, v in cols.items()}
    out["n"] = len(out["arrival"])
    out["tokens"] = tokens
    out["types"] = types
    return out


def single_batch(tr: dict, replica: int = 0) -> dict:
    """The sae_batch arrays of a single-replica trace."""
    out = {k: tr[k] for k in ("arrival", "prompt_off", "prompt_len", "decode_off", "decode_len",
                              "flags", "spb", "tokens", "types")}
    out["n"] = tr["n"]
    out["replica"] = np.full(tr["n"], replica, np.uint32)
    return out
