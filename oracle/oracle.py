"""ctypes binding of oracle/liboracle.so (test infrastructure only).

Marshals numpy arrays into the plain C functions of ``sae_oracle.cpp``.  No
arithmetic of the method lives here.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sae_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")

CXXFLAGS = ["-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC", "-pthread"]


def build(force: bool = False) -> str:
    """Compile the oracle (plain g++, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["g++", *CXXFLAGS, "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


class OrcParams(C.Structure):
    _fields_ = [("w", C.c_double * 5), ("alpha", C.c_double * 3), ("mu", C.c_double * 2),
                ("sigma", C.c_double * 2), ("gamma", C.c_double),
                ("eta", C.c_double), ("a_miss", C.c_double), ("b_reuse", C.c_double),
                ("T", C.c_double), ("beta_q", C.c_double), ("beta_ln", C.c_double),
                ("beta_gamma", C.c_double), ("learn_flags", C.c_uint32), ("mode", C.c_uint32)]


class OrcConfig(C.Structure):
    _fields_ = [("block_tokens", C.c_uint32), ("capacity", C.c_uint32),
                ("ghost_capacity", C.c_uint32), ("K", C.c_uint32),
                ("interval_ring", C.c_uint32), ("interval_keep", C.c_uint32),
                ("interval_min", C.c_uint32), ("n_bins", C.c_uint32),
                ("hash_seed", C.c_uint64), ("dt_eps", C.c_double), ("z_cut", C.c_double),
                ("init", OrcParams)]


class OrcTraj(C.Structure):
    _fields_ = [("E", C.c_uint64), ("request", C.c_uint64), ("w", C.c_double * 5),
                ("alpha", C.c_double * 3), ("mu", C.c_double * 2), ("sigma", C.c_double * 2),
                ("gamma", C.c_double)]


class OrcStats(C.Structure):
    _fields_ = [("requests", C.c_uint64), ("blocks_looked_up", C.c_uint64),
                ("hit_blocks", C.c_uint64), ("hit_tokens", C.c_uint64),
                ("prompt_tokens", C.c_uint64), ("evictions", C.c_uint64),
                ("evict_by_queue", C.c_uint64 * 4), ("evict_by_type", C.c_uint64 * 6),
                ("mae_by_type", C.c_uint64 * 6), ("learner_firings", C.c_uint64),
                ("eviction_rounds", C.c_uint64), ("blocks_scored", C.c_uint64),
                ("resident", C.c_uint64), ("resident_by_queue", C.c_uint64 * 4),
                ("E", C.c_uint64), ("next_id", C.c_uint64), ("gseq", C.c_uint64),
                ("now", C.c_double),
                ("ts_ev", C.c_uint64 * 5), ("ts_mae", C.c_uint64 * 5),
                ("ts_hit", C.c_uint64 * 5), ("ts_acc", C.c_uint64 * 5),
                ("qh", C.c_uint64 * 3), ("qe", C.c_uint64 * 3),
                ("pb_hit", C.c_uint64 * 16), ("pb_acc", C.c_uint64 * 16),
                ("iv_len", C.c_uint64 * 2)]


class OrcCharStats(C.Structure):
    _fields_ = [(k, C.c_uint64 * 6) for k in ("blocks", "reused", "later_blocks", "later_intra",
                                               "first_blocks", "first_inter")] + \
               [("pos_blocks", C.c_uint64 * 10), ("pos_reused", C.c_uint64 * 10),
                ("reuses_intra", C.c_uint64), ("reuses_inter", C.c_uint64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        # ORACLE_LIB: load a prebuilt copy instead (tests/test_oracle_mutations.py points it at
        # deliberately mutated builds to show that the pins catch one-line mistakes)
        L = C.CDLL(os.environ.get("ORACLE_LIB") or build())
        d, u32, u64, i32, vp = C.c_double, C.c_uint32, C.c_uint64, C.c_int, C.c_void_p
        P = C.POINTER
        sig = {
            "orc_ln": (d, [d]), "orc_exp": (d, [d]), "orc_erfc": (d, [d]),
            "orc_xxh64": (u64, [vp, u64, u64]),
            "orc_block_hash": (u64, [u64, vp, u32]),
            "orc_survival": (d, [d, d, d, d]),
            "orc_p_struct": (d, [u32, u32, d]),
            "orc_classify": (i32, [i32] * 6),
            "orc_tree_sum": (d, [vp, u64]),
            "orc_score": (d, [d, d, d, d]),
            "orc_priority": (d, [P(OrcParams), d, d, i32, i32, d, u32, u32]),
            "orc_create": (vp, [P(OrcConfig)]),
            "orc_destroy": (None, [vp]),
            "orc_set_params": (None, [vp, P(OrcParams)]),
            "orc_get_params": (None, [vp, P(OrcParams)]),
            "orc_admit": (i32, [vp, d, vp, vp, u32, vp, u32, u32, u32, vp, vp, u64, vp, vp, vp]),
            "orc_lookup": (i32, [vp, vp, vp, u32, vp, u32, vp]),
            "orc_evict": (i32, [vp, u64, d, vp, vp]),
            "orc_update": (None, [vp]),
            "orc_get_stats": (None, [vp, P(OrcStats)]),
            "orc_traj_count": (u64, [vp]),
            "orc_size": (u64, [vp]),
            "orc_traj_get": (None, [vp, vp]),
            "orc_intervals": (u64, [vp, i32, vp, u64]),
            "orc_resident": (u64, [vp, vp, vp, vp, vp, vp, vp, vp, vp, u64]),
            "orc_set_counters": (None, [vp, vp, vp, vp, vp, vp]),
            "orc_push_interval": (None, [vp, i32, d]),
            "orc_replay": (i32, [vp, u64] + [vp] * 9 + [vp, vp, u64, vp, vp, vp, vp]),
            "orc_characterize": (i32, [P(OrcConfig), u64] + [vp] * 10),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ---- pure functions -----------------------------------------------------------------
def ln(x): return lib().orc_ln(float(x))
def exp(x): return lib().orc_exp(float(x))
def erfc(x): return lib().orc_erfc(float(x))
def survival(dt, mu, sg, z_cut=30.0): return lib().orc_survival(dt, mu, sg, z_cut)
def p_struct(ob, omax, gam): return lib().orc_p_struct(int(ob), int(omax), float(gam))
def score(alpha, w, p, dt): return lib().orc_score(alpha, w, p, dt)
def priority(params: dict, q, tau, dt, ob=0, omax=1, dt_eps=1e-3, z_cut=30.0):
    """Eq.(1)-(3) of one block at elapsed time dt through the oracle's score()."""
    return lib().orc_priority(C.byref(make_params(params)), dt_eps, z_cut, int(q), int(tau),
                              float(dt), int(ob), int(omax))


def classify(tau, mt, ag, cid, is_struct, untempl):
    return lib().orc_classify(int(tau), int(mt), int(ag), int(cid), int(is_struct), int(untempl))


def xxh64(data: bytes, seed: int = 0) -> int:
    buf = np.frombuffer(data, dtype=np.uint8) if len(data) else np.zeros(1, np.uint8)
    return lib().orc_xxh64(_p(buf), len(data), seed)


def block_hash(prev: int, tokens) -> int:
    t = np.ascontiguousarray(tokens, dtype=np.uint32)
    return lib().orc_block_hash(prev, _p(t), len(t))


def tree_sum(y) -> float:
    a = np.ascontiguousarray(y, dtype=np.float64)
    return lib().orc_tree_sum(_p(a), len(a))


# ---- replica ------------------------------------------------------------------------
def make_params(p: dict) -> OrcParams:
    o = OrcParams()
    for k in ("w", "alpha", "mu", "sigma"):
        arr = getattr(o, k)
        for i, v in enumerate(p[k]):
            arr[i] = v
    for k in ("gamma", "eta", "a_miss", "b_reuse", "T", "beta_q", "beta_ln", "beta_gamma"):
        setattr(o, k, float(p[k]))
    o.learn_flags = int(p["learn_flags"])
    o.mode = int(p.get("mode", 0))
    return o


def params_dict(o: OrcParams) -> dict:
    return {"w": list(o.w), "alpha": list(o.alpha), "mu": list(o.mu), "sigma": list(o.sigma),
            "gamma": o.gamma, "eta": o.eta, "a_miss": o.a_miss, "b_reuse": o.b_reuse,
            "T": o.T, "beta_q": o.beta_q, "beta_ln": o.beta_ln, "beta_gamma": o.beta_gamma,
            "learn_flags": o.learn_flags, "mode": o.mode}


def make_config(cfg: dict) -> OrcConfig:
    c = OrcConfig()
    for k in ("block_tokens", "capacity", "ghost_capacity", "K", "interval_ring",
              "interval_keep", "interval_min", "n_bins"):
        setattr(c, k, int(cfg[k]))
    c.hash_seed = int(cfg["hash_seed"])
    c.dt_eps = float(cfg["dt_eps"])
    c.z_cut = float(cfg["z_cut"])
    c.init = make_params(cfg["params"])
    return c


@dataclass
class ReplayResult:
    out4: np.ndarray          # [n,4] hit_blocks, miss_blocks, matched_tokens, n_victims
    victims: np.ndarray       # u32 in eviction order
    voff: np.ndarray          # [n+1]
    hashes: np.ndarray | None
    taus: np.ndarray | None
    boff: np.ndarray          # [n+1]
    traj: list
    stats: OrcStats


class Replica:
    def __init__(self, cfg: dict):
        self.cfg = cfg
        self._c = make_config(cfg)
        self.h = lib().orc_create(C.byref(self._c))
        if not self.h:
            raise ValueError("invalid oracle config")

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_destroy(self.h)
            self.h = None

    def set_params(self, p: dict):
        lib().orc_set_params(self.h, C.byref(make_params(p)))

    def params(self) -> dict:
        o = OrcParams()
        lib().orc_get_params(self.h, C.byref(o))
        return params_dict(o)

    def stats(self) -> OrcStats:
        s = OrcStats()
        lib().orc_get_stats(self.h, C.byref(s))
        return s

    def size(self) -> int:
        """Number of resident blocks (cheap)."""
        return int(lib().orc_size(self.h))

    def traj(self) -> list:
        n = lib().orc_traj_count(self.h)
        arr = (OrcTraj * max(n, 1))()
        lib().orc_traj_get(self.h, arr)
        return [arr[i] for i in range(n)]

    def admit_req(self, now, ptok, ptyp, dtok, flags, spb):
        """Admit one request; returns (rc, res4, victims, hashes, taus)."""
        ptok = np.ascontiguousarray(ptok, np.uint32)
        ptyp = np.ascontiguousarray(ptyp, np.uint8)
        O = len(dtok)
        dbuf = np.ascontiguousarray(dtok if O else np.zeros(1, np.uint32), np.uint32)
        B = self.cfg["block_tokens"]
        nb = -(-len(ptok) // B) + -(-O // B)
        res4 = np.zeros(4, np.uint32)
        vcap = max(nb, 1) + 8
        vout = np.zeros(vcap, np.uint32)
        vn = np.zeros(1, np.uint64)
        hashes = np.zeros(max(nb, 1), np.uint64)
        taus = np.zeros(max(nb, 1), np.uint8)
        rc = lib().orc_admit(self.h, float(now), _p(ptok), _p(ptyp), len(ptok), _p(dbuf), O,
                             int(flags), int(spb), _p(res4), _p(vout), vcap, _p(vn),
                             _p(hashes), _p(taus))
        return rc, res4, vout[: int(vn[0])].copy(), hashes[:nb], taus[:nb]

    def lookup(self, ptok, ptyp, dtok) -> int:
        ptok = np.ascontiguousarray(ptok, np.uint32)
        ptyp = np.ascontiguousarray(ptyp, np.uint8)
        O = len(dtok)
        dbuf = np.ascontiguousarray(dtok if O else np.zeros(1, np.uint32), np.uint32)
        out = np.zeros(1, np.uint32)
        rc = lib().orc_lookup(self.h, _p(ptok), _p(ptyp), len(ptok), _p(dbuf), O, _p(out))
        if rc:
            raise ValueError("lookup rc=%d" % rc)
        return int(out[0])

    def evict(self, k, now):
        vout = np.zeros(max(k, 1), np.uint32)
        n = np.zeros(1, np.uint64)
        rc = lib().orc_evict(self.h, int(k), float(now), _p(vout), _p(n))
        return rc, vout[: int(n[0])].copy()

    def update(self):
        lib().orc_update(self.h)

    def intervals(self, s) -> np.ndarray:
        n = lib().orc_intervals(self.h, s, None, 0)
        out = np.zeros(max(n, 1), np.float64)
        lib().orc_intervals(self.h, s, _p(out), n)
        return out[:n]

    def resident(self) -> dict:
        n = lib().orc_resident(self.h, *([None] * 8), 0)
        cols = dict(hash=np.zeros(n, np.uint64), id=np.zeros(n, np.uint32),
                    last=np.zeros(n, np.float64), q=np.zeros(n, np.uint8),
                    tau=np.zeros(n, np.uint8), ntok=np.zeros(n, np.uint8),
                    ob=np.zeros(n, np.uint32), omax=np.zeros(n, np.uint32))
        lib().orc_resident(self.h, *[_p(cols[k]) for k in
                                     ("hash", "id", "last", "q", "tau", "ntok", "ob", "omax")], n)
        return cols

    def set_counters(self, ts=None, qh=None, qe=None, pbh=None, pba=None):
        conv = lambda a: None if a is None else np.ascontiguousarray(a, np.uint64)
        ts, qh, qe, pbh, pba = map(conv, (ts, qh, qe, pbh, pba))
        self._keep = (ts, qh, qe, pbh, pba)
        lib().orc_set_counters(self.h, _p(ts), _p(qh), _p(qe), _p(pbh), _p(pba))

    def push_interval(self, s, ln_dt):
        lib().orc_push_interval(self.h, s, float(ln_dt))

    def replay(self, tr, lo: int = 0, hi: int | None = None, want_hashes=True) -> ReplayResult:
        """Replay requests [lo, hi) of a single-replica trace dict (tracegen arrays)."""
        hi = tr["n"] if hi is None else hi
        n = hi - lo
        sl = slice(lo, hi)
        arr = {k: np.ascontiguousarray(tr[k][sl]) for k in
               ("arrival", "prompt_off", "prompt_len", "decode_off", "decode_len", "flags", "spb")}
        B = self.cfg["block_tokens"]
        nb = (-(-arr["prompt_len"].astype(np.int64) // B) - (-arr["decode_len"].astype(np.int64) // B))
        tot = int(nb.sum())
        out4 = np.zeros((n, 4), np.uint32)
        vcap = tot + 1
        vout = np.zeros(vcap, np.uint32)
        voff = np.zeros(n + 1, np.uint64)
        boff = np.zeros(n + 1, np.uint64)
        hashes = np.zeros(max(tot, 1), np.uint64) if want_hashes else None
        taus = np.zeros(max(tot, 1), np.uint8) if want_hashes else None
        rc = lib().orc_replay(self.h, n, _p(arr["arrival"]), _p(arr["prompt_off"]),
                              _p(arr["prompt_len"]), _p(arr["decode_off"]), _p(arr["decode_len"]),
                              _p(tr["tokens"]), _p(tr["types"]), _p(arr["flags"]), _p(arr["spb"]),
                              _p(out4), _p(vout), vcap, _p(voff), _p(hashes), _p(taus), _p(boff))
        if rc != 0:
            raise RuntimeError("oracle replay failed rc=%d" % rc)
        nv = int(voff[n])
        return ReplayResult(out4, vout[:nv].copy(), voff, None if hashes is None else hashes[:tot],
                            None if taus is None else taus[:tot], boff, self.traj(), self.stats())


def characterize(tr: dict, cfg: dict, single_turn=None) -> dict:
    """Characterisation pass (unbounded cache) of a single-replica trace: counters by token type,
    position bin and session locality (sae_oracle.cpp orc_characterize)."""
    c = make_config(cfg)
    st = single_turn if single_turn is not None else (~tr["continues"]).astype(np.uint8)
    arr = {k: np.ascontiguousarray(tr[k]) for k in ("prompt_off", "prompt_len", "decode_off", "decode_len")}
    sess = np.ascontiguousarray(tr["session"], np.uint32)
    turn = np.ascontiguousarray(tr["turn"], np.uint32)
    st = np.ascontiguousarray(st, np.uint8)
    o = OrcCharStats()
    rc = lib().orc_characterize(C.byref(c), tr["n"], _p(arr["prompt_off"]), _p(arr["prompt_len"]),
                                _p(arr["decode_off"]), _p(arr["decode_len"]), _p(tr["tokens"]),
                                _p(tr["types"]), _p(sess), _p(turn), _p(st), C.byref(o))
    if rc != 0:
        raise RuntimeError("oracle characterize rc=%d" % rc)
    return {k: (list(getattr(o, k)) if not isinstance(getattr(o, k), int) else getattr(o, k))
            for k, _ in OrcCharStats._fields_}


def point_mean_w(params: list, n_points: int) -> list:
    """mean_w sync, plain: for point p and type t, s = 0.0; s = s + w[p +
    n_points*i][t] for i in seed order; mean = s / S.  Returns new parameter dicts."""
    S = len(params) // n_points
    out = [dict(p, w=list(p["w"])) for p in params]
    for p in range(n_points):
        for t in range(5):
            s = 0.0
            for i in range(S):
                s = s + params[p + n_points * i]["w"][t]
            m = s / float(S)
            for i in range(S):
                out[p + n_points * i]["w"][t] = m
    return out
