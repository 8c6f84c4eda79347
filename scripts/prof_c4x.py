"""ncu helper: the c4x bench workload (2^24-block pool): prefill 600K requests (30 launches of
20000), then one 200-request launch (capture with -k regex:k_replay -s 30 -c 1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2605_18825_b200 import configs as C, sae as S
wl = bench.WORKLOADS["c4x"]
tr = bench.make_trace(wl, 0, n_requests=600_200)
pol = C.policy_config(tr["config"]["capacity"])
cache = S.SaeCache(pol["capacity"], policy=pol)
for lo in range(0, 600_000, 20000):
    cache.admit_batch(S.batch_to_torch(bench.slice_batch(tr, lo, lo + 20000)))
    torch.cuda.synchronize()
cache.admit_batch(S.batch_to_torch(bench.slice_batch(tr, 600_000, 600_200)))
torch.cuda.synchronize()
print("ok", cache.stats(0).requests, cache.stats(0).evictions)
