"""Oracle of the multi-turn session predictor (TEST INFRASTRUCTURE: only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference may use it).

Eq.(4):  y = W3 s(W2 s(W1 h + b1) + b2) + b3,  s = ReLU,  y_hat in {0, 1}
evaluated exactly as written, in fp64, from the bf16 / fp32 input values (decoded exactly).
The prediction is y > 0 (A45: the binary output thresholds the logit at 0).
Independent of csrc/: its own bf16 decoding, numpy matrix products as the library steps.
Pinned by tests/test_oracle_predictor.py (hand example tests/golden/predictor_hand.json,
linear-region matrix-chain identity, positive homogeneity, hidden-unit permutation
invariance, ReLU cut-off)."""
from __future__ import annotations

import numpy as np


def bf16_to_f64(bits) -> np.ndarray:
    """bf16 bit patterns -> their exact values (a bf16 is the upper half of an fp32)."""
    b = np.ascontiguousarray(bits, dtype=np.uint16).astype(np.uint32) << 16
    return b.view(np.float32).astype(np.float64)


def relu(x):
    return np.maximum(x, 0.0)


def predict_values(h, w1, b1, w2, b2, w3, b3):
    """Eq.(4) on decoded fp64 values: h [n, d], w1 [256, d], b1 [256], w2 [64, 256], b2 [64],
    w3 [64], b3 scalar.  Returns (y [n], y > 0)."""
    h = np.asarray(h, np.float64)
    a1 = relu(h @ np.asarray(w1, np.float64).T + np.asarray(b1, np.float64))   # s(W1 h + b1)
    a2 = relu(a1 @ np.asarray(w2, np.float64).T + np.asarray(b2, np.float64))  # s(W2 . + b2)
    y = a2 @ np.asarray(w3, np.float64) + float(b3)                            # W3 . + b3
    return y, y > 0.0


def predict(h_bits, W: dict):
    """Eq.(4) on the predgen layout: bf16 bit patterns for h, w1, w2; fp32 b1, b2, w3; b3."""
    return predict_values(bf16_to_f64(h_bits), bf16_to_f64(W["w1"]), W["b1"], bf16_to_f64(W["w2"]),
                          W["b2"], W["w3"], W["b3"])
