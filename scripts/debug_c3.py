"""Debug: replay the C3 trace prefix on the GPU and report the sticky error and select stats."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_18825_b200 import configs as C, tracegen as T, sae as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 6720
tr = T.make("c3", n_requests=n)
pol = C.policy_config(16384)
cache = S.SaeCache(16384, policy=pol)
b = S.batch_to_torch(T.single_batch(tr))
out = cache.admit_batch(b)
torch.cuda.synchronize()
try:
    cache.sync()
    print("no sticky error")
except Exception as e:
    print("sticky error:", e)
st = cache.stats(0) if False else None
from paper_2605_18825_b200.sae import lib, sae_replica_stats
import ctypes
s = sae_replica_stats()
rc = lib().sae_stats(cache.h, 0, ctypes.byref(s), None)
print("rc", rc, "requests", s.requests, "fail_seg", list(s.select_fail_seg), "passes", s.select_passes,
      "narrow", s.select_narrow, "cands", s.select_cands, "GP?")
