"""ncu helper: C2 (one single-CTA replica), 4 x 5000-request warm launches, then one
2000-request launch (capture with -k regex:k_replay -s 4 -c 1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_18825_b200 import configs as C, tracegen as T, sae as S
from bench import slice_batch
tr = T.make("c2", n_requests=22000)
pol = C.policy_config(tr["config"]["capacity"])
cache = S.SaeCache(pol["capacity"], policy=pol)
for lo in range(0, 20000, 5000):
    cache.admit_batch(S.batch_to_torch(slice_batch(tr, lo, lo + 5000)))
    torch.cuda.synchronize()
cache.admit_batch(S.batch_to_torch(slice_batch(tr, 20000, 22000)))
torch.cuda.synchronize()
print("ok", cache.stats(0).requests)
