"""Hand-traced golden micro-traces (tests/golden/*.json): loading and input building.

Each fixture is a short request sequence whose every expected value (victims, per-request
outputs, counters, learned parameters, intervals, trajectory) was derived BY HAND from the
cited passages of the paper and the DESIGN.md readings -- the derivation is written out in
the fixture.  This module only turns a fixture into the request arrays both sides consume;
it holds none of the method's arithmetic.  The oracle runs them in test_oracle_golden.py,
the CUDA path (through the C ABI) in test_gpu_golden.py.
"""
from __future__ import annotations

import copy
import glob
import json
import os

import numpy as np

from paper_2605_18825_b200 import configs as C

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def fixtures() -> list[dict]:
    out = []
    for p in sorted(glob.glob(os.path.join(GOLDEN, "*.json"))):
        d = json.load(open(p))
        if "ops" not in d:            # not a replay micro-trace (e.g. predictor_hand.json)
            continue
        d["_path"] = p
        out.append(d)
    return out


def policy(fx: dict) -> dict:
    c = fx["config"]
    p = copy.deepcopy(C.DEFAULT_PARAMS)
    p.update(c.get("params", {}))
    pol = C.policy_config(c["capacity"], K=c.get("K", 100), ghost_capacity=c.get("ghost_capacity"),
                          params=p)
    for k in ("interval_min", "interval_keep", "n_bins"):
        if k in c:
            pol[k] = c[k]
    return pol


def request_tokens(op: dict):
    """Block spec [[value, type(, ntok)], ...] -> prompt tokens u32, types u8.  Every token of
    a block carries the block's value (distinct values give distinct chained hashes) and its
    type (so tau = that type)."""
    toks, typs = [], []
    for blk in op["blocks"]:
        v, ty = int(blk[0]), int(blk[1])
        n = int(blk[2]) if len(blk) > 2 else 16
        toks.append(np.full(n, v, np.uint32))
        typs.append(np.full(n, ty, np.uint8))
    dec = [np.full(int(b[1]) if len(b) > 1 else 16, int(b[0]), np.uint32) for b in op.get("decode", [])]
    return (np.concatenate(toks), np.concatenate(typs),
            np.concatenate(dec) if dec else np.zeros(0, np.uint32))


def as_trace(ops: list[dict]) -> dict:
    """A run of admit ops as one single-replica trace (tracegen array layout)."""
    toks, typs, arr, po, pl, do, dl, fl, spb = [], [], [], [], [], [], [], [], []
    off = 0
    for op in ops:
        t, y, d = request_tokens(op)
        po.append(off); pl.append(len(t)); toks.append(t); typs.append(y); off += len(t)
        do.append(off); dl.append(len(d)); toks.append(d); typs.append(np.full(len(d), 5, np.uint8))
        off += len(d)
        arr.append(float(op["t"])); fl.append(int(op["flags"])); spb.append(int(op["spb"]))
    return {"n": len(ops), "arrival": np.array(arr, np.float64),
            "prompt_off": np.array(po, np.uint64), "prompt_len": np.array(pl, np.uint32),
            "decode_off": np.array(do, np.uint64), "decode_len": np.array(dl, np.uint32),
            "flags": np.array(fl, np.uint8), "spb": np.array(spb, np.uint32),
            "tokens": np.concatenate(toks) if toks else np.zeros(1, np.uint32),
            "types": np.concatenate(typs) if typs else np.zeros(1, np.uint8)}


def segments(fx: dict):
    """Split the op list into runs of consecutive admits and single evict/update ops."""
    run = []
    for op in fx["ops"]:
        if op["op"] == "admit":
            run.append(op)
            continue
        if run:
            yield ("admit", run)
            run = []
        yield (op["op"], op)
    if run:
        yield ("admit", run)


def check_value(name, got, want):
    """want: exact int / list, or [[value, abs_tol], ...] for floating point."""
    if isinstance(want, list) and want and isinstance(want[0], list):
        assert len(got) >= len(want), (name, got, want)
        for i, (v, tol) in enumerate(want):
            assert abs(float(got[i]) - v) <= tol, (name, i, float(got[i]), v, tol)
    elif isinstance(want, list):
        assert [int(x) for x in list(got)[: len(want)]] == want, (name, list(got), want)
    else:
        assert got == want, (name, got, want)
