"""Per-row bound on |y_kernel - y_exact| for the session predictor, derived from the
kernel's arithmetic (DESIGN.md "Session predictor" tolerance):
  GEMM1  d exact bf16 x bf16 products summed in fp32 (+ b1): |err| <= g(d+1) * S1
  ReLU   1-Lipschitz;  bf16 rounding of the GEMM2 operand: relative 2^-8
  GEMM2  256 exact bf16 products in fp32 (+ b2), propagated operand error
  layer3 64 fp32 multiply-adds (+ b3), propagated error
with g(k) = k u / (1 - k u) and u = 2^-23 (one fp32 ulp: holds for any rounding of the
tensor-core accumulator, round-to-nearest or truncation)."""
import numpy as np

from oracle import predictor as OP

U32 = 2.0 ** -23
UBF = 2.0 ** -8


def gamma(k):
    return k * U32 / (1 - k * U32)


def error_bound(h_bits, W):
    h = OP.bf16_to_f64(h_bits)
    w1, w2 = OP.bf16_to_f64(W["w1"]), OP.bf16_to_f64(W["w2"])
    b1, b2, w3 = (np.asarray(W[k], np.float64) for k in ("b1", "b2", "w3"))
    b3 = float(W["b3"])
    d = h.shape[1]
    z1 = h @ w1.T + b1
    e_z1 = gamma(d + 1) * (np.abs(h) @ np.abs(w1).T + np.abs(b1))
    a1 = np.maximum(z1, 0.0)
    e_a1 = e_z1 + UBF * (a1 + e_z1)
    z2 = a1 @ w2.T + b2
    e_z2 = e_a1 @ np.abs(w2).T + gamma(257) * ((a1 + e_a1) @ np.abs(w2).T + np.abs(b2))
    a2 = np.maximum(z2, 0.0)
    e_y = e_z2 @ np.abs(w3) + gamma(2 * 64 + 1) * ((a2 + e_z2) @ np.abs(w3) + abs(b3))
    return e_y + 1e-12 * (1.0 + a2 @ np.abs(w3))
