"""ncu helper: prefill a C4 replica (5 launches x 20000 requests), then one 200-request
launch (capture with -k regex:k_replay -s 5 -c 1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_18825_b200 import configs as C, tracegen as T, sae as S
from bench import slice_batch
tr = T.make("c4", n_requests=100200)
pol = C.policy_config(tr["config"]["capacity"])
cache = S.SaeCache(pol["capacity"], policy=pol)
for lo in range(0, 100000, 20000):
    cache.admit_batch(S.batch_to_torch(slice_batch(tr, lo, lo + 20000)))
    torch.cuda.synchronize()
cache.admit_batch(S.batch_to_torch(slice_batch(tr, 100000, 100200)))
torch.cuda.synchronize()
print("ok", cache.stats(0).requests)
