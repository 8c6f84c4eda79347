"""Profile helper: warm a C2 replica with 2500 requests, then one 500-request batch
(the launch ncu captures with -k regex:k_replay -s 1 -c 1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_18825_b200 import configs as C, tracegen as T, sae as S
from bench import slice_batch
wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
n_warm, n_prof = 2500, 500
tr = T.make(wl, n_requests=n_warm + n_prof)
pol = C.policy_config(tr["config"]["capacity"])
cache = S.SaeCache(pol["capacity"], policy=pol)
for lo, hi in ((0, n_warm), (n_warm, n_warm + n_prof)):
    b = S.batch_to_torch(slice_batch(tr, lo, hi))
    cache.admit_batch(b)
    torch.cuda.synchronize()
print("done", cache.stats(0).requests)
st = cache.stats(0)
print("chunks~", st.learner_firings, "passes", st.select_passes, "cands/pass", st.select_cands / max(st.select_passes, 1),
      "big", st.select_big, "fails", list(st.select_fail_seg), "evictions", st.evictions, "rounds", st.eviction_rounds)
print("phase ms", [round(x / 1e6, 1) for x in st.phase_ns])
