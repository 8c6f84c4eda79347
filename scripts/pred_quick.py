"""Quick timing of the session predictor kernel (CUDA events, L2 > flushed by input size)."""
import sys
import numpy as np
import torch
from paper_2605_18825_b200 import predgen as PG
from paper_2605_18825_b200 import sae as S

d = 4096
n = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 17)
W = PG.weights(d)
h = torch.randn(n, d, device="cuda").to(torch.bfloat16).view(torch.int16)
P = S.SessionPredictor(W["w1"], W["b1"], W["w2"], W["b2"], W["w3"], W["b3"])
y = torch.empty(n, dtype=torch.float32, device="cuda")
for _ in range(3):
    P.predict(h, logit=y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
K = 20
e0.record()
for _ in range(K):
    P.predict(h, logit=y)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / K
by = n * d * 2
fl = 2.0 * n * (d * 256 + 256 * 64 + 64)
print("n=%d d=%d: %.3f ms/launch  %.1f M pred/s  %.0f GB/s (h)  %.0f TFLOP/s" % (n, d, ms, n / ms / 1e3, by / ms / 1e6, fl / ms / 1e9))
