"""compute-sanitizer driver: C1 replay (single CTA) + a small multi-CTA group replay."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_18825_b200 import configs as C, tracegen as T, sae as S
from bench import slice_batch
tr = T.make("c1")
pol = C.policy_config(64, K=8)
cache = S.SaeCache(64, policy=pol, traj_capacity=256)
cache.admit_batch(S.batch_to_torch(T.single_batch(tr)), want_hashes=True)
cache.lookup(S.batch_to_torch(T.single_batch(tr)))
cache.evict(0, 5, float(tr["arrival"][-1]) + 1)
cache.update()
torch.cuda.synchronize()
print("c1 ok", cache.stats(0).evictions)
tr2 = T.generate(C.get("c3", n_requests=300, seed=7)); T.materialize(tr2)
pol2 = C.policy_config(4500, K=50)
c2 = S.SaeCache(4500, policy=pol2, ctas_per_replica=3)
c2.admit_batch(S.batch_to_torch(T.single_batch(tr2)))
torch.cuda.synchronize()
print("group ok", c2.stats(0).evictions)
