"""Thin Python binding of libsae.so (include/sae.h): argument marshalling only.

Every step of the hot path runs in the CUDA kernels of ``csrc/sae.cu``; this
module only converts torch tensors to device pointers and C structs.  There is
no CPU fallback: importing it on a box without the built extension (or calling
it without a CUDA device) raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

from . import configs as CFG

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SAE_LIB_PATH") or os.path.join(_HERE, "libsae.so")   # override: debug builds

SAE_ABI_VERSION = 3
ERRORS = {0: "SAE_OK", -1: "SAE_E_INVAL", -2: "SAE_E_CAPACITY_ZERO", -3: "SAE_E_EMPTY",
          -4: "SAE_E_NOT_RESIDENT", -5: "SAE_E_TIME", -6: "SAE_E_OVERFLOW", -7: "SAE_E_OOM",
          -8: "SAE_E_CUDA", -9: "SAE_E_ABI", -10: "SAE_E_INTERNAL"}


class SaeError(RuntimeError):
    def __init__(self, status, msg=""):
        super().__init__("%s (%d) %s" % (ERRORS.get(status, "?"), status, msg))
        self.status = status


class sae_params(C.Structure):
    _fields_ = [("w", C.c_double * 5), ("alpha", C.c_double * 3), ("mu", C.c_double * 2),
                ("sigma", C.c_double * 2), ("gamma", C.c_double), ("eta", C.c_double),
                ("a_miss", C.c_double), ("b_reuse", C.c_double), ("T", C.c_double),
                ("beta_q", C.c_double), ("beta_ln", C.c_double), ("beta_gamma", C.c_double),
                ("learn_flags", C.c_uint32), ("mode", C.c_uint32)]


class sae_config(C.Structure):
    _fields_ = [("abi_version", C.c_uint32), ("block_tokens", C.c_uint32),
                ("capacity_blocks", C.c_uint32), ("n_replicas", C.c_uint32),
                ("ghost_capacity", C.c_uint32), ("K", C.c_uint32), ("interval_ring", C.c_uint32),
                ("interval_keep", C.c_uint32), ("interval_min", C.c_uint32),
                ("n_pos_bins", C.c_uint32), ("ctas_per_replica", C.c_uint32),
                ("traj_capacity", C.c_uint32), ("hash_seed", C.c_uint64), ("dt_eps", C.c_double),
                ("z_cut", C.c_double), ("init", sae_params), ("device", C.c_int32),
                ("_pad", C.c_uint32)]


class sae_batch(C.Structure):
    _fields_ = [("n", C.c_uint32), ("_pad", C.c_uint32), ("total_blocks", C.c_uint64)] + \
               [(k, C.c_void_p) for k in ("replica", "arrival", "prompt_off", "prompt_len",
                                          "decode_off", "decode_len", "tokens", "types", "flags",
                                          "shared_prefix_blocks")]


class sae_admit_out(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in ("hit_blocks", "miss_blocks", "matched_tokens",
                                          "n_victims", "victim_off", "victim_ids")] + \
               [("victim_cap", C.c_uint64), ("block_hash", C.c_void_p), ("block_tau", C.c_void_p)]


class sae_replica_stats(C.Structure):
    _fields_ = [("requests", C.c_uint64), ("blocks_looked_up", C.c_uint64),
                ("hit_blocks", C.c_uint64), ("hit_tokens", C.c_uint64),
                ("prompt_tokens", C.c_uint64), ("evictions", C.c_uint64),
                ("evict_by_queue", C.c_uint64 * 4), ("evict_by_type", C.c_uint64 * 6),
                ("mae_by_type", C.c_uint64 * 6), ("learner_firings", C.c_uint64),
                ("eviction_rounds", C.c_uint64), ("blocks_scored", C.c_uint64),
                ("blocks_scored_struct", C.c_uint64),
                ("resident", C.c_uint64), ("resident_by_queue", C.c_uint64 * 4),
                ("E", C.c_uint64), ("next_id", C.c_uint64), ("gseq", C.c_uint64),
                ("now", C.c_double), ("ts_ev", C.c_uint64 * 5), ("ts_mae", C.c_uint64 * 5),
                ("ts_hit", C.c_uint64 * 5), ("ts_acc", C.c_uint64 * 5), ("qh", C.c_uint64 * 3),
                ("qe", C.c_uint64 * 3), ("pb_hit", C.c_uint64 * 16), ("pb_acc", C.c_uint64 * 16),
                ("iv_len", C.c_uint64 * 2), ("traj_count", C.c_uint64),
                ("select_passes", C.c_uint64), ("select_cands", C.c_uint64),
                ("select_big", C.c_uint64), ("select_fail_seg", C.c_uint64 * 10),
                ("phase_ns", C.c_uint64 * 16),
                ("select_narrow", C.c_uint64), ("select_raw", C.c_uint64),
                ("params", sae_params), ("stage2_chunks", C.c_uint64)]


class sae_char_stats(C.Structure):
    _fields_ = [(k, C.c_uint64 * 6) for k in ("blocks", "reused", "later_blocks", "later_intra",
                                               "first_blocks", "first_inter")] + \
               [("pos_blocks", C.c_uint64 * 10), ("pos_reused", C.c_uint64 * 10),
                ("reuses_intra", C.c_uint64), ("reuses_inter", C.c_uint64)]


class sae_predictor_config(C.Structure):
    _fields_ = [("abi_version", C.c_uint32), ("d", C.c_uint32), ("device", C.c_int32), ("_pad", C.c_uint32)]


class sae_traj(C.Structure):
    _fields_ = [("E", C.c_uint64), ("request", C.c_uint64), ("w", C.c_double * 5),
                ("alpha", C.c_double * 3), ("mu", C.c_double * 2), ("sigma", C.c_double * 2),
                ("gamma", C.c_double)]


class sae_layout_info(C.Structure):
    _fields_ = [(k, C.c_uint32) for k in ("threads", "ctas_per_replica", "ctas_per_sm", "chunks",
                                          "cand_global", "coresident")]


EXPORTS = ["sae_create", "sae_destroy", "sae_set_params", "sae_params_gather", "sae_params_scatter",
           "sae_batch_blocks", "sae_admit_batch", "sae_admit_batch_host", "sae_lookup", "sae_evict", "sae_update",
           "sae_stats", "sae_get_traj", "sae_sync", "sae_last_error", "sae_gen_tokens",
           "sae_launch_count", "sae_profile", "sae_profile_read", "sae_params_point_mean",
           "sae_counters_device", "sae_priority", "sae_profile_read_hash", "sae_characterize",
           "sae_select", "sae_predictor_create", "sae_predictor_destroy", "sae_predict", "sae_predictor_launch_count",
           "sae_predictor_last_error", "sae_layout"]

# sae_counters (include/sae.h): field order of the whole-ctx counter totals
COUNTER_FIELDS = (["requests", "blocks_looked_up", "hit_blocks", "hit_tokens", "prompt_tokens",
                   "evictions"] + ["evict_by_queue%d" % i for i in range(4)] +
                  ["evict_by_type%d" % i for i in range(6)] + ["mae_by_type%d" % i for i in range(6)] +
                  ["learner_firings", "eviction_rounds", "blocks_scored", "blocks_scored_struct"])

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError("libsae.so not built (run __graft_entry__.build()); no CPU fallback")
        L = C.CDLL(LIB_PATH)
        vp, u32, u64, i32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int
        P = C.POINTER
        sig = {
            "sae_create": (i32, [P(sae_config), P(vp)]),
            "sae_destroy": (i32, [vp]),
            "sae_set_params": (i32, [vp, u32, P(sae_params), vp]),
            "sae_params_gather": (i32, [vp, vp, vp]),
            "sae_params_scatter": (i32, [vp, vp, vp]),
            "sae_batch_blocks": (i32, [vp, P(sae_batch), P(u64), vp]),
            "sae_admit_batch": (i32, [vp, P(sae_batch), P(sae_admit_out), vp]),
            "sae_admit_batch_host": (i32, [vp, P(sae_batch), u64, u64, vp, vp, P(sae_admit_out),
                                           P(u64), P(u64), vp]),
            "sae_lookup": (i32, [vp, P(sae_batch), vp, vp]),
            "sae_evict": (i32, [vp, u32, u32, C.c_double, vp, vp, vp]),
            "sae_select": (i32, [vp, u32, u32, C.c_double, u32, vp, vp, vp]),
            "sae_update": (i32, [vp, u32, vp]),
            "sae_stats": (i32, [vp, u32, P(sae_replica_stats), vp]),
            "sae_get_traj": (i32, [vp, u32, vp, u64, P(u64), vp]),
            "sae_sync": (i32, [vp, vp]),
            "sae_last_error": (C.c_char_p, [vp]),
            "sae_gen_tokens": (i32, [u64, u64, vp, vp, vp, vp, vp, vp, vp, vp]),
            "sae_launch_count": (u64, [vp]),
            "sae_profile": (i32, [vp, i32]),
            "sae_params_point_mean": (i32, [vp, u32, u32, vp, vp]),
            "sae_profile_read": (i32, [vp, P(C.c_double), P(u64)]),
            "sae_profile_read_hash": (i32, [vp, P(C.c_double), P(u64)]),
            "sae_characterize": (i32, [vp, P(sae_batch), vp, vp, vp, P(sae_char_stats), vp]),
            "sae_counters_device": (i32, [vp, vp, vp]),
            "sae_priority": (i32, [P(sae_params), C.c_double, C.c_double, u64] + [vp] * 7),
            "sae_predictor_create": (i32, [P(sae_predictor_config), vp, vp, vp, vp, vp, C.c_float, P(vp)]),
            "sae_predictor_destroy": (i32, [vp]),
            "sae_predict": (i32, [vp, vp, u32, vp, vp, vp, vp]),
            "sae_predictor_launch_count": (u64, [vp]),
            "sae_predictor_last_error": (C.c_char_p, [vp]),
            "sae_layout": (i32, [vp, P(sae_layout_info)]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _lib = L
    return _lib


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def make_params(p: dict) -> sae_params:
    o = sae_params()
    for k in ("w", "alpha", "mu", "sigma"):
        arr = getattr(o, k)
        for i, v in enumerate(p[k]):
            arr[i] = v
    for k in ("gamma", "eta", "a_miss", "b_reuse", "T", "beta_q", "beta_ln", "beta_gamma"):
        setattr(o, k, float(p[k]))
    o.learn_flags = int(p["learn_flags"])
    o.mode = int(p.get("mode", 0))
    return o


def params_dict(o: sae_params) -> dict:
    return {"w": list(o.w), "alpha": list(o.alpha), "mu": list(o.mu), "sigma": list(o.sigma),
            "gamma": o.gamma, "eta": o.eta, "a_miss": o.a_miss, "b_reuse": o.b_reuse, "T": o.T,
            "beta_q": o.beta_q, "beta_ln": o.beta_ln, "beta_gamma": o.beta_gamma,
            "learn_flags": o.learn_flags, "mode": o.mode}


# torch dtypes carrying the C unsigned layouts bit for bit
_TD = {"replica": torch.int32, "arrival": torch.float64, "prompt_off": torch.int64,
       "prompt_len": torch.int32, "decode_off": torch.int64, "decode_len": torch.int32,
       "tokens": torch.int32, "types": torch.uint8, "flags": torch.uint8, "spb": torch.int32}
_NPD = {"replica": np.uint32, "arrival": np.float64, "prompt_off": np.uint64,
        "prompt_len": np.uint32, "decode_off": np.uint64, "decode_len": np.uint32,
        "tokens": np.uint32, "types": np.uint8, "flags": np.uint8, "spb": np.uint32}


def batch_to_torch(b: dict, device="cuda", pin: bool = False, block_tokens: int = 16) -> dict:
    """numpy sae_batch arrays (tracegen layout) -> torch tensors (device or pinned host);
    total_blocks is counted with the ctx's block size (the device re-checks it)."""
    out = {}
    for k, td in _TD.items():
        a = np.ascontiguousarray(b[k], dtype=_NPD[k])
        t = torch.from_numpy(a.view({np.uint32: np.int32, np.uint64: np.int64}.get(a.dtype.type, a.dtype)))
        if pin:
            out[k] = t.pin_memory()
        else:
            out[k] = t.to(device, non_blocking=False)
    out["n"] = int(b["n"])
    out["block_tokens"] = B = int(block_tokens)
    pl = np.asarray(b["prompt_len"], np.int64)
    dl = np.asarray(b["decode_len"], np.int64)
    out["total_blocks"] = int((-(-pl // B) - (-dl // B)).sum())
    return out


class SaeCache:
    """One sae_ctx: R independent replicas of the SAECache block pool on one GPU."""

    def __init__(self, capacity: int, n_replicas: int = 1, K: int = 100,
                 ghost_capacity: int | None = None, params: dict | None = None,
                 traj_capacity: int = 0, device: int | None = None, policy: dict | None = None,
                 ctas_per_replica: int = 0):
        if not torch.cuda.is_available():
            raise SaeError(-8, "no CUDA device (the SAECache path has no CPU fallback)")
        pc = policy or CFG.policy_config(capacity, K=K, ghost_capacity=ghost_capacity, params=params)
        self.policy = pc
        self.device = torch.cuda.current_device() if device is None else device
        c = sae_config()
        c.abi_version = SAE_ABI_VERSION
        c.block_tokens = pc["block_tokens"]
        c.capacity_blocks = pc["capacity"]
        c.n_replicas = n_replicas
        c.ghost_capacity = pc["ghost_capacity"]
        c.K = pc["K"]
        c.interval_ring = pc["interval_ring"]
        c.interval_keep = pc["interval_keep"]
        c.interval_min = pc["interval_min"]
        c.n_pos_bins = pc["n_bins"]
        c.ctas_per_replica = ctas_per_replica
        c.traj_capacity = traj_capacity
        c.hash_seed = pc["hash_seed"]
        c.dt_eps = pc["dt_eps"]
        c.z_cut = pc["z_cut"]
        c.init = make_params(pc["params"])
        c.device = self.device
        self._cfg = c
        self.R = n_replicas
        self.h = C.c_void_p()
        self._check(lib().sae_create(C.byref(c), C.byref(self.h)))

    def _check(self, rc):
        if rc != 0:
            msg = lib().sae_last_error(self.h).decode() if self.h else ""
            raise SaeError(rc, msg)

    def close(self):
        if self.h:
            lib().sae_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- calls ---------------------------------------------------------------------
    def _batch(self, b: dict) -> sae_batch:
        if b.get("block_tokens", 16) != self.policy["block_tokens"]:
            raise SaeError(-1, "batch counted with %d-token blocks, ctx uses %d (batch_to_torch("
                           "block_tokens=...))" % (b.get("block_tokens", 16), self.policy["block_tokens"]))
        sb = sae_batch()
        sb.n = b["n"]
        sb.total_blocks = b["total_blocks"]
        for k, f in (("replica", "replica"), ("arrival", "arrival"), ("prompt_off", "prompt_off"),
                     ("prompt_len", "prompt_len"), ("decode_off", "decode_off"),
                     ("decode_len", "decode_len"), ("tokens", "tokens"), ("types", "types"),
                     ("flags", "flags"), ("spb", "shared_prefix_blocks")):
            setattr(sb, f, b[k].data_ptr())
        return sb

    def alloc_out(self, b: dict, want_hashes: bool = False) -> dict:
        n, tb = b["n"], b["total_blocks"]
        dev = b["arrival"].device
        o = {k: torch.empty(n, dtype=torch.int32, device=dev)
             for k in ("hit_blocks", "miss_blocks", "matched_tokens", "n_victims")}
        o["victim_off"] = torch.empty(n + 1, dtype=torch.int64, device=dev)
        o["victim_ids"] = torch.empty(max(tb, 1), dtype=torch.int32, device=dev)
        if want_hashes:
            o["block_hash"] = torch.empty(max(tb, 1), dtype=torch.int64, device=dev)
            o["block_tau"] = torch.empty(max(tb, 1), dtype=torch.uint8, device=dev)
        return o

    def admit_batch(self, b: dict, out: dict | None = None, want_hashes: bool = False, stream=None):
        out = out if out is not None else self.alloc_out(b, want_hashes)
        ao = sae_admit_out()
        for k in ("hit_blocks", "miss_blocks", "matched_tokens", "n_victims", "victim_off", "victim_ids"):
            setattr(ao, k, out[k].data_ptr())
        ao.victim_cap = out["victim_ids"].numel()
        ao.block_hash = out["block_hash"].data_ptr() if "block_hash" in out else None
        ao.block_tau = out["block_tau"].data_ptr() if "block_tau" in out else None
        self._keep = (b, out)
        self._check(lib().sae_admit_batch(self.h, C.byref(self._batch(b)), C.byref(ao), _stream(stream)))
        return out

    def admit_batch_host(self, hb: dict, tok_h, typ_h, tok_d, typ_d, a: int, z: int, stream=None):
        """End-to-end call through the C ABI's sae_admit_batch_host: the step's request arrays
        (pinned host tensors in hb) and the token arena range [a, z) (pinned tok_h / typ_h)
        are copied host->device by the library, the batch is replayed, and the per-request
        outputs and victim ids come back into pinned host buffers (valid after the stream
        synchronises).  Successive calls pipeline (the library stages inputs in two slots on
        its own copy stream): the outputs alternate between two pinned sets, so a call's
        results stay valid while the next call runs.  Returns (host outputs, h2d bytes,
        d2h bytes)."""
        n, tb = hb["n"], hb["total_blocks"]
        st = self._staging = getattr(self, "_staging", {"slot": 0})
        slot = st["slot"]
        st["slot"] ^= 1
        hout = st.get(slot)
        if hout is None or hout["victim_ids"].numel() < max(tb, 1) or hout["hit_blocks"].numel() < n:
            if hout is not None:
                self.sync(stream)           # the set may still be a target of a queued copy
            hout = st[slot] = {k: torch.empty(max(2 * n, 1), dtype=torch.int32, pin_memory=True)
                               for k in ("hit_blocks", "miss_blocks", "matched_tokens", "n_victims")}
            hout["victim_off"] = torch.empty(2 * n + 1, dtype=torch.int64, pin_memory=True)
            hout["victim_ids"] = torch.empty(max(2 * tb, 1), dtype=torch.int32, pin_memory=True)
        sb = sae_batch()
        sb.n = n
        sb.total_blocks = tb
        for k, f in (("replica", "replica"), ("arrival", "arrival"), ("prompt_off", "prompt_off"),
                     ("prompt_len", "prompt_len"), ("decode_off", "decode_off"),
                     ("decode_len", "decode_len"), ("flags", "flags"), ("spb", "shared_prefix_blocks")):
            setattr(sb, f, hb[k].data_ptr())
        sb.tokens = tok_h.data_ptr()
        sb.types = typ_h.data_ptr()
        ao = sae_admit_out()
        for k in ("hit_blocks", "miss_blocks", "matched_tokens", "n_victims", "victim_off", "victim_ids"):
            setattr(ao, k, hout[k].data_ptr())
        ao.victim_cap = hout["victim_ids"].numel()
        h2d, d2h = C.c_uint64(), C.c_uint64()
        st["keep%d" % slot] = (hb, hout)        # host inputs stay alive while their copies are queued
        self._check(lib().sae_admit_batch_host(self.h, C.byref(sb), a, z, tok_d.data_ptr(),
                                               typ_d.data_ptr(), C.byref(ao), C.byref(h2d),
                                               C.byref(d2h), _stream(stream)))
        res = {k: v[: n] for k, v in hout.items() if k not in ("victim_off", "victim_ids")}
        res["victim_off"] = hout["victim_off"][: n + 1]
        res["victim_ids"] = hout["victim_ids"][: max(tb, 1)]
        return res, h2d.value, d2h.value

    def lookup(self, b: dict, stream=None) -> torch.Tensor:
        hit = torch.empty(b["n"], dtype=torch.int32, device=b["arrival"].device)
        self._check(lib().sae_lookup(self.h, C.byref(self._batch(b)), hit.data_ptr(), _stream(stream)))
        return hit

    def evict(self, replica: int, k: int, now: float, stream=None):
        ids = torch.empty(max(k, 1), dtype=torch.int32, device="cuda")
        n = torch.zeros(1, dtype=torch.int32, device="cuda")
        self._check(lib().sae_evict(self.h, replica, k, float(now), ids.data_ptr(), n.data_ptr(),
                                    _stream(stream)))
        return ids, n

    def select(self, replica: int, m: int, now: float, passes: int = 1, vids: torch.Tensor | None = None,
               n_out: torch.Tensor | None = None, stream=None):
        """Read-only fused score/select (sae_select): the ids of the next m victims."""
        if vids is None:
            vids = torch.empty(max(m, 1), dtype=torch.int32, device="cuda")
        if n_out is None:
            n_out = torch.zeros(1, dtype=torch.int32, device="cuda")
        self._check(lib().sae_select(self.h, replica, m, now, passes, _ptr(vids), _ptr(n_out), _stream(stream)))
        return vids, n_out

    def update(self, replica: int | None = None, stream=None):
        r = 0xFFFFFFFF if replica is None else replica
        self._check(lib().sae_update(self.h, r, _stream(stream)))

    def set_params(self, replica: int, p: dict, stream=None):
        self._check(lib().sae_set_params(self.h, replica, C.byref(make_params(p)), _stream(stream)))

    def params_gather(self, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """All replicas' sae_params as a [R, sizeof/8] float64 device tensor."""
        nd = C.sizeof(sae_params) // 8
        if out is None:
            out = torch.empty((self.R, nd), dtype=torch.float64, device="cuda")
        self._check(lib().sae_params_gather(self.h, out.data_ptr(), _stream(stream)))
        return out

    def params_scatter(self, t: torch.Tensor, stream=None):
        self._check(lib().sae_params_scatter(self.h, t.data_ptr(), _stream(stream)))

    def stats(self, replica: int = 0, stream=None) -> sae_replica_stats:
        s = sae_replica_stats()
        self._check(lib().sae_stats(self.h, replica, C.byref(s), _stream(stream)))
        return s

    def traj(self, replica: int = 0, stream=None) -> list:
        n = C.c_uint64()
        lib().sae_get_traj(self.h, replica, None, 0, C.byref(n), _stream(stream))
        arr = (sae_traj * max(n.value, 1))()
        self._check(lib().sae_get_traj(self.h, replica, arr, n.value, C.byref(n), _stream(stream)))
        return [arr[i] for i in range(n.value)]

    def counters_device(self, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """[len(COUNTER_FIELDS)] int64 device tensor: every replica's additive counters summed
        on the device (for an NCCL int64 all-reduce across ranks)."""
        if out is None:
            out = torch.empty(len(COUNTER_FIELDS), dtype=torch.int64, device="cuda")
        self._check(lib().sae_counters_device(self.h, out.data_ptr(), _stream(stream)))
        return out

    def characterize(self, b: dict, session, turn, single_turn, stream=None) -> dict:
        """Characterisation pass (sae_characterize) of the batch b (device tensors, one trace
        in arrival order) with per-request session / turn (int32) and single_turn (uint8)
        device tensors; returns the counters as a dict of lists / ints."""
        o = sae_char_stats()
        sb = sae_batch()
        sb.n = b["n"]
        sb.total_blocks = b["total_blocks"]
        for k, f in (("arrival", "arrival"), ("prompt_off", "prompt_off"), ("prompt_len", "prompt_len"),
                     ("decode_off", "decode_off"), ("decode_len", "decode_len"), ("tokens", "tokens"),
                     ("types", "types"), ("flags", "flags"), ("spb", "shared_prefix_blocks")):
            setattr(sb, f, b[k].data_ptr())
        self._check(lib().sae_characterize(self.h, C.byref(sb), session.data_ptr(), turn.data_ptr(),
                                           single_turn.data_ptr(), C.byref(o), _stream(stream)))
        return {k: (list(getattr(o, k)) if not isinstance(getattr(o, k), int) else getattr(o, k))
                for k, _ in sae_char_stats._fields_}

    def sync(self, stream=None):
        self._check(lib().sae_sync(self.h, _stream(stream)))

    def layout(self) -> dict:
        """sae_layout: threads per CTA, CTAs per replica / per SM, co-resident CTAs, replay
        chunks per replica run (task-split persistent replay when > 1), candidate buffer place."""
        o = sae_layout_info()
        self._check(lib().sae_layout(self.h, C.byref(o)))
        return {k: int(getattr(o, k)) for k, _ in o._fields_}

    def launches(self) -> int:
        return int(lib().sae_launch_count(self.h))

    def profile(self, enable: bool = True):
        self._check(lib().sae_profile(self.h, 1 if enable else 0))

    def profile_read_hash(self):
        """(summed K1 hashing-kernel ms, number of its launches) since the last read."""
        ms = C.c_double()
        n = C.c_uint64()
        self._check(lib().sae_profile_read_hash(self.h, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def profile_read(self):
        """(summed replay-kernel ms, number of replay launches) since the last read."""
        ms = C.c_double()
        n = C.c_uint64()
        self._check(lib().sae_profile_read(self.h, C.byref(ms), C.byref(n)))
        return ms.value, n.value


def params_point_mean(all_params: torch.Tensor, n_points: int, stream=None) -> torch.Tensor:
    """mean_w over seeds per parameter point (fixed order), on the device."""
    out = torch.empty_like(all_params)
    rc = lib().sae_params_point_mean(all_params.data_ptr(), all_params.shape[0], n_points,
                                     out.data_ptr(), _stream(stream))
    if rc != 0:
        raise SaeError(rc, "sae_params_point_mean")
    return out


def priority(params: dict, q, tau, dt, ob, omax, dt_eps: float = 1e-3, z_cut: float = 30.0,
             stream=None) -> torch.Tensor:
    """Eq.(1)-(3) on the device (sae_priority): device tensors q u8, tau u8, dt f64, ob / omax
    i32 of one length -> P f64 (NaN for EF), the select's arithmetic exactly."""
    out = torch.empty_like(dt)
    rc = lib().sae_priority(C.byref(make_params(params)), float(dt_eps), float(z_cut), dt.numel(),
                            q.data_ptr(), tau.data_ptr(), dt.data_ptr(), ob.data_ptr(), omax.data_ptr(),
                            out.data_ptr(), _stream(stream))
    if rc != 0:
        raise SaeError(rc, "sae_priority")
    return out


def gen_tokens(seed: int, pieces: dict, dst: np.ndarray, n_tokens: int, device="cuda",
               stream=None):
    """K7: materialise a trace's tokens/types on the device from its piece table."""
    st = torch.from_numpy(pieces["stream"].view(np.int64)).to(device)
    sa = torch.from_numpy(pieces["start"].astype(np.int64)).to(device)
    ln = torch.from_numpy(pieces["len"].astype(np.uint32).view(np.int32)).to(device)
    ds = torch.from_numpy(dst.astype(np.int64)).to(device)
    ty = torch.from_numpy(pieces["type"].astype(np.uint8)).to(device)
    tokens = torch.empty(max(n_tokens, 1), dtype=torch.int32, device=device)
    types = torch.empty(max(n_tokens, 1), dtype=torch.uint8, device=device)
    rc = lib().sae_gen_tokens(seed, len(pieces["len"]), st.data_ptr(), sa.data_ptr(), ln.data_ptr(),
                              ds.data_ptr(), ty.data_ptr(), tokens.data_ptr(), types.data_ptr(),
                              _stream(stream))
    if rc != 0:
        raise SaeError(rc, "sae_gen_tokens")
    return tokens, types


class SessionPredictor:
    """Multi-turn session predictor, Eq.(4), on the tensor cores (csrc/predictor.cu).

    Weights as produced by ``predgen.weights`` (host numpy): w1 / w2 bf16 bit patterns
    (uint16), b1 / b2 / w3 float32, b3 a float.  ``predict`` takes the hidden states as a
    CUDA tensor of bf16 (or their uint16 bit patterns) shaped [n, d]."""

    def __init__(self, w1, b1, w2, b2, w3, b3, device: int | None = None):
        L = lib()
        if not torch.cuda.is_available():
            raise RuntimeError("SessionPredictor needs a CUDA device (no CPU fallback)")
        w1 = np.ascontiguousarray(w1, np.uint16)
        self.d = int(w1.shape[1])
        cfg = sae_predictor_config()
        cfg.abi_version, cfg.d = SAE_ABI_VERSION, self.d
        cfg.device = torch.cuda.current_device() if device is None else device
        self._keep = [w1, np.ascontiguousarray(b1, np.float32), np.ascontiguousarray(w2, np.uint16),
                      np.ascontiguousarray(b2, np.float32), np.ascontiguousarray(w3, np.float32)]
        h = C.c_void_p()
        rc = L.sae_predictor_create(C.byref(cfg), *[a.ctypes.data_as(C.c_void_p) for a in self._keep],
                                    C.c_float(float(b3)), C.byref(h))
        if rc != 0:
            raise SaeError(rc, L.sae_predictor_last_error(None).decode())
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().sae_predictor_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def predict(self, hidden: torch.Tensor, rows: torch.Tensor | None = None, logit: torch.Tensor | None = None,
                flags: torch.Tensor | None = None, stream=None):
        """logit [n] float32 (allocated when neither logit nor flags is given) and/or flags
        (uint8, bit 0 := prediction), indexed by rows (int32) when given."""
        assert hidden.is_cuda and hidden.dim() == 2 and hidden.shape[1] == self.d and hidden.is_contiguous()
        n = int(hidden.shape[0])
        if logit is None and flags is None:
            logit = torch.empty(n, dtype=torch.float32, device=hidden.device)
        rc = lib().sae_predict(self.h, C.c_void_p(hidden.data_ptr()), n, _ptr(rows), _ptr(logit), _ptr(flags),
                               _stream(stream))
        if rc != 0:
            raise SaeError(rc, lib().sae_predictor_last_error(self.h).decode())
        return logit

    def launches(self) -> int:
        return int(lib().sae_predictor_launch_count(self.h))
