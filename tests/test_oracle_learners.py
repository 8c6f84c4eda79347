"""Learner pins (SURVEY c.7 L1-L4): closed forms, library statistics, clamps."""
import math

import numpy as np

import oracle
from paper_2605_18825_b200 import configs as C


def replica(**pover):
    p = dict(C.DEFAULT_PARAMS)
    p.update(pover)
    return oracle.Replica(C.policy_config(64, params=p))


def ts_counters(ev, mae, hit, acc):
    return [ev] * 5 + [mae] * 5 + [hit] * 5 + [acc] * 5


def test_token_weight_additive_closed_form():
    # w0=1, eta=0.1, r_miss=r_reuse=1, a=5, b=2: 0.9*1 + 0.1*8 = 1.7000000000000002
    R = replica(w=[1.0] * 5, learn_flags=C.L_TOKENS)
    R.set_counters(ts=ts_counters(100, 100, 100, 100))
    R.update()
    p = R.params()
    assert p["w"] == [1.7000000000000002] * 5
    st = R.stats()
    assert list(st.ts_ev) == [99] * 5 and list(st.ts_acc) == [99] * 5   # floor(99x/100)


def test_token_weight_threshold_and_fixed_point():
    R = replica(w=[2.0] * 5, learn_flags=C.L_TOKENS)
    R.set_counters(ts=ts_counters(10, 10, 10, 10))      # evicted must be > 10
    R.update()
    assert R.params()["w"] == [2.0] * 5
    # r_miss = r_reuse = 0 -> target 1: |w - 1| = 0.9^n after n updates
    R = replica(w=[2.0] * 5, learn_flags=C.L_TOKENS)
    for n in range(200):
        R.set_counters(ts=ts_counters(1000, 0, 0, 1000))
        R.update()
    w = R.params()["w"][0]
    assert abs((w - 1.0) - 0.9 ** 200) < 1e-12


def test_token_weight_multiplicative_rule():
    # Alg. P:725: w <- w (1 + eta * miss_rate)
    R = replica(w=[1.0] * 5, learn_flags=C.L_TOKENS | C.L_TOKEN_MULT)
    R.set_counters(ts=ts_counters(100, 50, 0, 0))
    R.update()
    assert R.params()["w"] == [1.0 * (1.0 + 0.1 * 0.5)] * 5


def test_queue_weight_alg_closed_form():
    # hits 20, evictions 10, T 2, beta 0.3, alpha0 1 -> 1.3
    R = replica(learn_flags=C.L_QUEUES)
    R.set_counters(qh=[20, 0, 20], qe=[10, 10, 5])
    R.update()
    a = R.params()["alpha"]
    assert a[0] == 1.3
    assert a[1] == 1.0            # hits 0 -> target 1 -> stays 1
    assert a[2] == 1.0            # evictions must be > 5
    st = R.stats()
    assert list(st.qh) == [0, 0, 0] and list(st.qe) == [0, 0, 0]   # reset


def test_queue_weight_never_below_one_under_alg_rule():
    rng = np.random.default_rng(3)
    R = replica(learn_flags=C.L_QUEUES)
    for _ in range(500):
        R.set_counters(qh=rng.integers(0, 50, 3), qe=rng.integers(0, 50, 3))
        R.update()
        a = R.params()["alpha"]
        assert all(1.0 <= x <= 3.0 for x in a)   # consequence of tgt >= 1 (A19)


def test_lognormal_closed_forms():
    R = replica(mu=[0.0, 0.0], sigma=[1.0, 1.0], beta_ln=1.0, learn_flags=C.L_LOGNORMAL)
    for _ in range(21):
        R.push_interval(0, 2.0)
    for _ in range(20):
        R.push_interval(1, 5.0)
    R.update()
    p = R.params()
    assert p["mu"][0] == 2.0 and p["sigma"][0] == 0.1     # sd = 0 -> floor 0.1
    assert p["mu"][1] == 0.0 and p["sigma"][1] == 1.0     # n <= 20 -> no update
    assert len(R.intervals(1)) == 20
    for _ in range(300):
        R.push_interval(1, 1.0)
    R.update()
    assert len(R.intervals(1)) == 200                    # truncate to last 200


def test_adaptive_beta_closed_forms():
    """Adaptive EMA factor (reading A28): rho = mean (x - mu)^2 / sigma^2 over the
    ln-intervals; rho > 1 -> beta doubled (at most 1), else halved."""
    F = C.L_LOGNORMAL | C.L_ADAPTIVE_BETA
    # observations exactly at the model mean: rho = 0 -> beta 0.15: mu stays, sigma 1 -> 0.85
    R = replica(mu=[2.0, 2.0], sigma=[1.0, 1.0], beta_ln=0.3, learn_flags=F)
    for _ in range(21):
        R.push_interval(0, 2.0)
    R.update()
    p = R.params()
    assert p["mu"][0] == 2.0 and abs(p["sigma"][0] - 0.85) < 1e-15
    # without the flag the same update uses beta 0.3: sigma -> 0.7
    R = replica(mu=[2.0, 2.0], sigma=[1.0, 1.0], beta_ln=0.3, learn_flags=C.L_LOGNORMAL)
    for _ in range(21):
        R.push_interval(0, 2.0)
    R.update()
    assert abs(R.params()["sigma"][0] - 0.7) < 1e-15
    # observations 3 sigma away: rho = 9 -> beta 0.6: mu 2 -> 2 + 0.6 x 3 = 3.8, sigma -> 0.4
    R = replica(mu=[2.0, 2.0], sigma=[1.0, 1.0], beta_ln=0.3, learn_flags=F)
    for _ in range(21):
        R.push_interval(1, 5.0)
    R.update()
    p = R.params()
    assert abs(p["mu"][1] - 3.8) < 1e-15 and abs(p["sigma"][1] - 0.4) < 1e-15
    # beta 0.7 doubled is capped at 1: jump to the sample statistics (sigma floor 0.1)
    R = replica(mu=[2.0, 2.0], sigma=[1.0, 1.0], beta_ln=0.7, learn_flags=F)
    for _ in range(21):
        R.push_interval(0, 6.0)
    R.update()
    p = R.params()
    assert p["mu"][0] == 6.0 and p["sigma"][0] == 0.1


def test_lognormal_statistics_vs_numpy():
    rng = np.random.default_rng(4)
    x = rng.normal(4.82, 1.25, 1000)
    R = replica(mu=[0.0, 0.0], sigma=[0.0, 0.0], beta_ln=1.0, learn_flags=C.L_LOGNORMAL)
    for v in x:
        R.push_interval(0, v)
    R.update()
    p = R.params()
    assert abs(p["mu"][0] - np.mean(x)) <= 1e-14 * abs(np.mean(x))
    assert abs(p["sigma"][0] - np.std(x)) <= 1e-13 * np.std(x)   # population std (A24)


def test_lognormal_round_trip_on_lognormal_draws():
    # 20k log-normal(4.82, 1.25) draws -> (mu, sigma) within +-0.05
    rng = np.random.default_rng(5)
    t = rng.lognormal(4.82, 1.25, 20000)
    R = replica(mu=[0.0, 0.0], sigma=[0.0, 0.0], beta_ln=1.0, learn_flags=C.L_LOGNORMAL)
    R2 = oracle.Replica(dict(C.policy_config(64, params=R.params()), interval_ring=20000))
    for v in t:
        R2.push_interval(0, oracle.ln(v))
    R2.update()
    p = R2.params()
    assert abs(p["mu"][0] - 4.82) < 0.05 and abs(p["sigma"][0] - 1.25) < 0.05


def test_decay_power_closed_forms():
    # ratio 0.9 -> est = 1/(0.9+0.1) = 1.0
    R = replica(gamma=2.0, beta_gamma=1.0, learn_flags=C.L_DECAY)
    R.set_counters(pbh=[100] * 5 + [90] * 5, pba=[100] * 10)
    R.update()
    assert abs(R.params()["gamma"] - 1.0) <= 4e-16
    # ratio 0 -> est 10 -> clamp to 3.0
    R = replica(gamma=1.0, beta_gamma=1.0, learn_flags=C.L_DECAY)
    R.set_counters(pbh=[100] * 5 + [0] * 5, pba=[100] * 10)
    R.update()
    assert R.params()["gamma"] == 3.0
    # a half without data -> no update
    R = replica(gamma=1.7, beta_gamma=1.0, learn_flags=C.L_DECAY)
    R.set_counters(pbh=[5] * 10, pba=[10] * 5 + [0] * 5)
    R.update()
    assert R.params()["gamma"] == 1.7


def test_clamp_fuzz_all_learners():
    rng = np.random.default_rng(6)
    R = replica(learn_flags=C.L_DEFAULT)
    for _ in range(3000):
        ev = rng.integers(0, 1000, 5)
        R.set_counters(ts=list(ev) + list(rng.integers(0, ev + 1)) +
                       list(rng.integers(0, 100, 5)) + list(rng.integers(0, 200, 5)),
                       qh=rng.integers(0, 1000, 3), qe=rng.integers(0, 100, 3),
                       pbh=rng.integers(0, 50, 10), pba=rng.integers(50, 100, 10))
        for s in (0, 1):
            for v in rng.normal(2.0, 3.0, rng.integers(0, 30)):
                R.push_interval(s, v)
        R.update()
        p = R.params()
        assert all(0.1 <= w <= 5.0 for w in p["w"])
        assert all(0.1 <= a <= 3.0 for a in p["alpha"])
        assert all(s >= 0.1 for s in p["sigma"])
        assert 0.3 <= p["gamma"] <= 3.0
        assert all(math.isfinite(v) for v in p["mu"])


def test_relative_queue_rule_equal_efficiency():
    # P:816 with E_q / E_bar = 1 -> (1)^(1/T) = exp(ln(1)/T) = 1
    R = replica(alpha=[2.0, 2.0, 2.0], learn_flags=C.L_QUEUES | C.L_QUEUE_RELATIVE)
    # empty cache: capacity fractions 0 -> E_q undefined -> no update, counters reset
    R.set_counters(qh=[5, 5, 5], qe=[9, 9, 9])
    R.update()
    assert R.params()["alpha"] == [2.0, 2.0, 2.0]
    assert list(R.stats().qh) == [0, 0, 0]
