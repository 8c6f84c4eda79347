"""Pins of the session-predictor oracle (oracle/predictor.py, Eq.(4)) against what
the definition and mathematics fix -- a hand-worked example, the linear-region matrix-chain
identity, positive homogeneity, hidden-unit permutation invariance, the ReLU cut-off -- and
of the bf16 encoding of the input generator."""
import json
import os

import numpy as np

from oracle import predictor as OP
from paper_2605_18825_b200 import predgen as PG

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "predictor_hand.json")


def _rand_net(rng, d=48, n1=256, n2=64, nonneg=False):
    f = (lambda *s: rng.uniform(0.0, 1.0, s)) if nonneg else (lambda *s: rng.normal(0.0, 1.0, s))
    return f(n1, d) / np.sqrt(d), f(n1), f(n2, n1) / 16.0, f(n2), f(n2) / 8.0, float(f(1)[0])


def test_hand_example():
    g = json.load(open(GOLDEN))
    y, p = OP.predict_values(np.array(g["h"]), np.array(g["w1"]), g["b1"], np.array(g["w2"]), g["b2"],
                             g["w3"], g["b3"])
    assert list(y) == g["y"]
    assert list(p) == g["pred"]


def test_linear_region_equals_matrix_chain():
    # all inputs and weights >= 0: no ReLU is active, so Eq.(4) is the affine map
    # y = (W3 W2 W1) h + (W3 W2) b1 + W3 b2 + b3, evaluated here in the other association
    rng = np.random.default_rng(1)
    w1, b1, w2, b2, w3, b3 = _rand_net(rng, nonneg=True)
    h = rng.uniform(0.0, 1.0, (17, 48))
    y, _ = OP.predict_values(h, w1, b1, w2, b2, w3, b3)
    m32 = w3 @ w2
    ref = h @ (m32 @ w1) + m32 @ b1 + w3 @ b2 + b3
    assert np.allclose(y, ref, rtol=1e-12, atol=0)


def test_positive_homogeneity_exact():
    # ReLU networks are positively homogeneous in (h, biases): scaling by 2 is exact in binary
    rng = np.random.default_rng(2)
    w1, b1, w2, b2, w3, b3 = _rand_net(rng)
    h = rng.normal(0, 1, (33, 48))
    y, _ = OP.predict_values(h, w1, b1, w2, b2, w3, b3)
    y2, _ = OP.predict_values(2 * h, w1, 2 * b1, w2, 2 * b2, w3, 2 * b3)
    assert np.array_equal(y2, 2 * y)


def test_hidden_unit_permutation_invariance():
    rng = np.random.default_rng(3)
    w1, b1, w2, b2, w3, b3 = _rand_net(rng)
    h = rng.normal(0, 1, (9, 48))
    y, p = OP.predict_values(h, w1, b1, w2, b2, w3, b3)
    p1, p2 = rng.permutation(256), rng.permutation(64)
    yq, pq = OP.predict_values(h, w1[p1], b1[p1], w2[p2][:, p1], b2[p2], w3[p2], b3)
    assert np.allclose(yq, y, rtol=1e-12, atol=1e-12)
    # a transposed / mismatched permutation (a plausible indexing slip) changes the output
    yb, _ = OP.predict_values(h, w1[p1], b1, w2[p2][:, p1], b2[p2], w3[p2], b3)
    assert not np.allclose(yb, y)


def test_relu_cutoff():
    rng = np.random.default_rng(4)
    w1, b1, w2, b2, w3, b3 = _rand_net(rng)
    h = rng.normal(0, 1, (5, 48))
    y, _ = OP.predict_values(h, w1, np.full(256, -1e6), w2, b2, w3, b3)
    assert np.allclose(y, np.full(5, w3 @ np.maximum(b2, 0) + b3), rtol=1e-14, atol=0)
    assert np.ptp(y) == 0.0      # every row reduces to the same constant


def test_bf16_encoding_roundtrip():
    x = np.array([1.0, -2.5, 0.0, 3.140625, 1.0 + 2.0 ** -8, 1.0 + 3 * 2.0 ** -8, 65504.0], np.float32)
    bits = PG.to_bf16_bits(x)
    assert list(bits[:4]) == [0x3F80, 0xC020, 0x0000, 0x4049]
    # ties to even: 1 + 2^-8 -> 1.0 (0x3F80); 1 + 3*2^-8 -> 1 + 2^-6 (0x3F82)
    assert bits[4] == 0x3F80 and bits[5] == 0x3F82
    assert list(OP.bf16_to_f64(bits)[:4]) == [1.0, -2.5, 0.0, 3.140625]


def test_generator_shapes_and_scale():
    W = PG.weights(d=256, seed=7)
    assert W["w1"].shape == (256, 256) and W["w2"].shape == (64, 256) and W["w3"].shape == (64,)
    w1 = OP.bf16_to_f64(W["w1"])
    assert np.abs(w1).max() <= 1 / 16 * (1 + 2 ** -8)
    h = PG.hidden(10, 256, seed=3)
    assert h.dtype == np.uint16 and h.shape == (10, 256)
    assert np.array_equal(h, PG.hidden(10, 256, seed=3))
