"""Stress run: R replicas of the C5 pool, N requests from S seeds, per-replica learner points.

Usage: python scripts/repro_c5.py R N S P  (P=1: point r%32);  no args: a fixed sweep in subprocesses.
Used to chase the CTA-barrier drift documented in DESIGN.md."""
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1:
    import numpy as np, torch
    from paper_2605_18825_b200 import configs as C, tracegen as T, sae as S, replicas as RP
    R, n, nseeds, sp = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    traces = []
    for sd in range(nseeds):
        t = T.generate(C.get("c5", n_requests=n), seed=0x5AEC1000 + sd); T.materialize(t); traces.append(t)
    cache = S.SaeCache(2304, n_replicas=R, policy=C.policy_config(2304))
    if sp:
        for r in range(R):
            cache.set_params(r, C.c5_point_params(r % 32 if sp == 1 else sp))
    batch = T.replicate(traces, [(r // 32) % nseeds for r in range(R)])
    out = cache.admit_batch(S.batch_to_torch(batch))
    torch.cuda.synchronize()
    print("OK", R, n, cache.stats(0).requests, cache.stats(0).evictions, flush=True)
else:
    for args in [("32", "10000", "1", "1"), ("32", "3000", "1", "1"), ("256", "2000", "8", "1"), ("64", "10000", "2", "1"), ("160", "10000", "5", "1")]:
        r = subprocess.run([sys.executable, __file__, *args], capture_output=True, text=True, timeout=600)
        print(args, r.stdout.strip()[-200:], r.stderr.strip()[-300:] if r.returncode else "", flush=True)
