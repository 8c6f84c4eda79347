"""Pins of the oracle's feedback side against hand-traced golden micro-traces
(tests/golden/*.json, each with its citation and its derivation written out).

These fix what no closed form covers: the ghost FIFO (expiry, the tau credited on a
miss-after-evict), eviction accounting and the K-crossing chunk whose later victims use
the new parameters, the hit / access / bin / interval statistics credited to the old
queue, orphan refresh, the relative queue rule with all three E_q defined (and with one
undefined), the queue / type / (mu, sigma) / position routing of Eq.(1)-(3), and the full
Alg.1 Classify truth table.  tests/test_oracle_mutations.py shows that a one-line mistake
in each of these oracle functions fails one of them."""
import os

import numpy as np
import pytest

import oracle
from tests.golden_traces import GOLDEN, check_value, fixtures, policy, request_tokens

FIX = fixtures()


def run_oracle(fx):
    R = oracle.Replica(policy(fx))
    for op in fx["ops"]:
        if op["op"] == "admit":
            t, y, d = request_tokens(op)
            rc, res, vic, _, _ = R.admit_req(op["t"], t, y, d, op["flags"], op["spb"])
            assert rc == 0, (fx["name"], op)
            if "out" in op:
                assert [int(x) for x in res] == op["out"], (fx["name"], op["t"], list(res), op["out"])
            if "victims" in op:
                assert [int(v) for v in vic] == op["victims"], (fx["name"], op["t"], list(vic), op["victims"])
        elif op["op"] == "evict":
            rc, vic = R.evict(op["k"], op["t"])
            assert rc == op.get("rc", 0)
            assert [int(v) for v in vic] == op["victims"], (fx["name"], list(vic), op["victims"])
        elif op["op"] == "update":
            R.update()
    return R


@pytest.mark.parametrize("fx", FIX, ids=[f["name"] for f in FIX])
def test_golden_trace(fx):
    R = run_oracle(fx)
    st = R.stats()
    for k, want in fx.get("stats", {}).items():
        got = getattr(st, k)
        check_value(k, list(got) if not isinstance(got, (int, float)) else got, want)
    par = R.params()
    for k, want in fx.get("params", {}).items():
        check_value(k, par[k], want)
    for s, want in fx.get("intervals", {}).items():
        iv = R.intervals(int(s))
        assert len(iv) == len(want), (s, iv, want)
        check_value("iv%s" % s, iv, want)
    if "traj" in fx:
        tj = R.traj()
        assert len(tj) == len(fx["traj"])
        for a, w in zip(tj, fx["traj"]):
            assert a.E == w["E"] and a.request == w["request"]
            check_value("traj.alpha", list(a.alpha), w["alpha"])


def classify_table():
    rows = []
    for line in open(os.path.join(GOLDEN, "classify_table.txt")):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        *bits, q = line.split()
        rows.append(([int(b) for b in bits], {"EF": 0, "CHAT": 1, "AGENT": 2, "STRUCT": 3}[q]))
    return rows


def test_classify_full_truth_table():
    rows = classify_table()
    assert len(rows) == 192
    for (tau, mt, ag, cid, st, un), q in rows:
        assert oracle.classify(tau, mt, ag, cid, st, un) == q, (tau, mt, ag, cid, st, un, q)
