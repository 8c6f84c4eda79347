"""Seeded synthetic inputs of the session predictor (Eq.(4)): hidden states and
weights.  Input generation only -- none of the method's arithmetic lives here (the oracle and
the CUDA path both consume these arrays).

* Hidden states: the paper feeds the final-layer hidden state of the last prompt token of a
  history-free request.  No serving model runs here, so h is synthetic: i.i.d.
  N(0, 1) per channel (the scale of a normed final layer), rounded to bf16 (A44).
* Weights: the paper's trained predictor is not available; W1 (256 x d), W2 (64 x 256), W3
  (1 x 64) and the biases are drawn like torch.nn.Linear's default initialisation,
  U(-1/sqrt(fan_in), 1/sqrt(fan_in)); W1 and W2 are rounded to bf16, the rest stay fp32.
bf16 values are carried as their uint16 bit patterns (round to nearest even from fp32)."""
from __future__ import annotations

import numpy as np

N1, N2 = 256, 64          # hidden widths
D_DEFAULT = 4096          # d: "roughly one million parameters" / "4 MB"; A43


def to_bf16_bits(x) -> np.ndarray:
    """fp32 -> bf16 bit patterns, round to nearest even (finite inputs)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def weights(d: int = D_DEFAULT, seed: int = 0x5AEC2000) -> dict:
    rng = np.random.default_rng(seed)

    def lin(fan_out, fan_in):
        k = 1.0 / np.sqrt(fan_in)
        return (rng.uniform(-k, k, (fan_out, fan_in)).astype(np.float32),
                rng.uniform(-k, k, fan_out).astype(np.float32))

    w1, b1 = lin(N1, d)
    w2, b2 = lin(N2, N1)
    w3, b3 = lin(1, N2)
    return {"w1": to_bf16_bits(w1), "b1": b1, "w2": to_bf16_bits(w2), "b2": b2, "w3": w3[0],
            "b3": float(b3[0]), "d": d}


def hidden(n: int, d: int = D_DEFAULT, seed: int = 0x5AEC2001) -> np.ndarray:
    """[n, d] bf16 bit patterns of synthetic last-token hidden states."""
    rng = np.random.default_rng(seed)
    out = np.empty((n, d), np.uint16)
    step = max(1, (1 << 24) // max(d, 1))
    for i in range(0, n, step):            # bounded temporaries for large n
        j = min(n, i + step)
        out[i:j] = to_bf16_bits(rng.standard_normal((j - i, d), dtype=np.float32))
    return out
