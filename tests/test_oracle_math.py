"""Pins for the oracle's arithmetic against things other than
itself: mpmath at 50 digits, closed forms, and the paper's stated constants."""
import math
import struct

import mpmath
import numpy as np
import pytest

import oracle

mpmath.mp.dps = 50


def ulps(a: float, b: float) -> int:
    ia = struct.unpack("<q", struct.pack("<d", a))[0]
    ib = struct.unpack("<q", struct.pack("<d", b))[0]
    return abs(ia - ib)


def rnd(x) -> float:
    return float(mpmath.mpf(x))


@pytest.fixture(scope="module")
def rng():
    return np.random.default_rng(12345)


def test_ln_within_one_ulp_of_mpmath(rng):
    # dt in [1e-3, 1e7] (the replay's range, SURVEY c.7) + wide random + edges
    xs = list(np.exp(rng.uniform(np.log(1e-3), np.log(1e7), 3000)))
    xs += list(np.exp(rng.uniform(-700, 700, 1000)))
    xs += [1e-3, 0.5, 1.0 - 2**-53, 1.0 + 2**-52, 2.0, 1.5, 0.75, 1e7, 5e-324, 1.7976931348623157e308]
    for x in xs:
        want = rnd(mpmath.log(mpmath.mpf(float(x))))
        assert ulps(oracle.ln(x), want) <= 1, x
    assert oracle.ln(1.0) == 0.0
    assert math.isinf(oracle.ln(0.0)) and oracle.ln(0.0) < 0
    assert math.isnan(oracle.ln(-1.0))


def test_exp_within_one_ulp_of_mpmath(rng):
    xs = list(rng.uniform(-745, 709, 3000)) + list(rng.uniform(-2, 2, 1000))
    xs += [0.0, 1e-30, -1e-30, 0.34657359027997264, 0.5, -0.5, 1.0397207708399179, 709.7, -745.0]
    for x in xs:
        want = rnd(mpmath.exp(mpmath.mpf(float(x))))
        got = oracle.exp(x)
        if want < 2.2250738585072014e-308:  # subnormal results: absolute check
            assert abs(got - want) <= 5e-324 * 2, x
        else:
            assert ulps(got, want) <= 1, x
    assert oracle.exp(0.0) == 1.0
    assert math.isinf(oracle.exp(710.0))
    assert oracle.exp(-746.0) == 0.0


def test_erfc_within_one_ulp_of_mpmath(rng):
    # z/sqrt2 for z in [-40, 40] (SURVEY c.7) and every fdlibm branch boundary
    xs = list(rng.uniform(-40 / math.sqrt(2), 40 / math.sqrt(2), 3000))
    xs += list(rng.uniform(-1.5, 1.5, 1000))
    xs += [0.0, 1e-20, 0.25, 0.84375, -0.84375, 1.25, -1.25, 1 / 0.35, -1 / 0.35, 6.0, -6.0,
           27.9, 28.0, -28.0]
    # fdlibm's erfc composes two exp() calls and a division in the tail, so its
    # final error is bounded by a few ulp (not 1): pin <= 3 ulp everywhere and
    # <= 1 ulp on >= 97% of points.  A wrong coefficient shows up as >> 3 ulp.
    big = 0
    for x in xs:
        want = rnd(mpmath.erfc(mpmath.mpf(float(x))))
        got = oracle.erfc(x)
        if want < 2.2250738585072014e-308:
            assert abs(got - want) <= 1e-320, x
        else:
            e = ulps(got, want)
            assert e <= 3, (x, got, want)
            big += e > 1
    assert big <= 0.03 * len(xs)


def test_survival_closed_forms():
    # Eq.(1): S(e^mu) = 1 - Phi(0) = 0.5
    for mu, sg in [(4.82, 1.25), (2.28, 1.34), (4.15, 0.97), (0.0, 1.0)]:
        assert ulps(oracle.survival(math.exp(mu), mu, sg), 0.5) <= 2
    # SURVEY c.7 values (checked with scipy; S:201's 0.487 is wrong)
    assert abs(oracle.survival(110.6, 4.82, 1.25) - 0.536358560478409) < 1e-15
    assert abs(oracle.survival(453.6, 2.28, 1.34) - 0.00209432357897181) < 1e-17
    # independent: 1 - Phi via mpmath ncdf
    for dt, mu, sg in [(1.0, 4.82, 1.25), (10.0, 2.28, 1.34), (1e5, 4.15, 0.97), (1e-3, 2.28, 1.34)]:
        z = (mpmath.log(dt) - mu) / sg
        want = rnd(1 - mpmath.ncdf(z))
        # tail is ill-conditioned in z (d ln S / dz ~ z), so compare relatively
        assert abs(oracle.survival(dt, mu, sg) - want) <= 1e-13 * want


def test_survival_monotone_and_cutoff():
    dts = np.exp(np.linspace(np.log(1e-3), np.log(1e7), 20001))
    for mu, sg in [(4.82, 1.25), (2.28, 1.34), (4.15, 0.1)]:
        s = np.array([oracle.survival(d, mu, sg) for d in dts])
        assert np.all(np.diff(s) <= 0)
    # z > z_cut -> exactly 0; just below -> positive
    mu, sg = 0.0, 0.1
    assert oracle.survival(math.exp(3.01), mu, sg) == 0.0
    assert oracle.survival(math.exp(2.99), mu, sg) > 0.0


def test_p_struct_closed_forms():
    # Eq.(2)
    assert oracle.p_struct(0, 7, 1.3) == 1.0
    for omax in (1, 2, 7, 100, 4095):
        for g in (0.3, 1.0, 2.7):
            assert oracle.p_struct(omax, omax, g) == 0.0
    for omax in (3, 10, 97):
        for ob in range(omax + 1):
            assert ulps(oracle.p_struct(ob, omax, 1.0), 1.0 - ob / omax) <= 1
    # (o/omax)^gamma against mpmath
    for ob, omax, g in [(1, 3, 0.5), (5, 9, 2.2), (33, 100, 0.94)]:
        want = rnd(1 - mpmath.power(mpmath.mpf(ob) / omax, g))
        assert abs(oracle.p_struct(ob, omax, g) - want) <= 4 * np.spacing(want)


def test_score_eq3():
    # alpha=1, w=1, p=0.5, dt=2 -> 0.25 exactly
    assert oracle.score(1.0, 1.0, 0.5, 2.0) == 0.25
    assert oracle.score(2.0, 1.5, 0.25, 0.5) == 1.5


def test_tree_sum(rng):
    for n in (1, 2, 3, 7, 20, 21, 200, 1000, 4096):
        x = rng.normal(3.0, 2.0, n)
        assert abs(oracle.tree_sum(x) - math.fsum(x)) <= 1e-13 * max(1.0, abs(math.fsum(x)))
        # padding-independence: explicit zero padding to 4x gives identical bits
        y = np.concatenate([x, np.zeros(3 * n)])
        assert oracle.tree_sum(y) == oracle.tree_sum(x)
    # exact on small integers
    assert oracle.tree_sum(np.arange(100, dtype=float)) == 4950.0


def test_classify_cascade_alg1():
    Q_EF, Q_CHAT, Q_AGENT, Q_STRUCT = 0, 1, 2, 3
    # Alg.1, hand cases
    assert oracle.classify(4, 1, 1, 1, 1, 0) == Q_EF      # cot -> evict-first
    assert oracle.classify(5, 1, 0, 0, 0, 0) == Q_EF      # decode -> evict-first
    assert oracle.classify(0, 0, 0, 0, 0, 1) == Q_EF      # untemplated -> evict-first
    assert oracle.classify(1, 1, 1, 0, 0, 0) == Q_AGENT   # multi-turn agentic
    assert oracle.classify(3, 1, 0, 0, 1, 0) == Q_CHAT    # multi-turn chat
    assert oracle.classify(3, 0, 0, 1, 1, 0) == Q_CHAT    # conversation id non-empty
    assert oracle.classify(0, 0, 1, 1, 0, 0) == Q_CHAT    # agentic but predicted single, cid
    assert oracle.classify(1, 0, 0, 0, 1, 0) == Q_STRUCT  # shared prefix
    assert oracle.classify(0, 0, 0, 0, 0, 0) == Q_STRUCT  # system prompt
    assert oracle.classify(2, 0, 1, 0, 0, 0) == Q_EF      # fallthrough
