"""Baselines and ablation ladder on the GPU: every variant of
paper_2605_18825_b200.ablation.variants() x S seeds of a synthetic workload as replicas of one
sae_ctx, replayed side by side; reports token / block hit rate and the TTFT model's prefill
tokens per variant, relative to LRU, and the learned parameters.

    python scripts/ablation.py [--workload c5|c2|c4s] [--seeds 32] [--requests 10000] [--out gpurun_out/ablation]

The directions to compare with the paper: SAECache above LRU/LFU, the learner
ladder improving step by step from Fixed-Param, Fixed-Param degrading when the
mix differs from the chat-fitted one."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2605_18825_b200 import ablation as A
from paper_2605_18825_b200 import configs as C
from paper_2605_18825_b200 import sae as S
from paper_2605_18825_b200 import tracegen as T

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c5", help="c5 (balanced), c2 (multi-turn-dominant), c4s (single-turn-dominant)")
ap.add_argument("--seeds", type=int, default=32)
ap.add_argument("--requests", type=int, default=10_000)
ap.add_argument("--out", default="gpurun_out/ablation")
a = ap.parse_args()

mix = {"c5": C.MIX_BAL, "c2": C.MIX_MT, "c4s": C.MIX_ST}[a.workload]
traces = []
for sd in range(a.seeds):
    t = T.generate(C.get("c5", n_requests=a.requests, mix=mix), seed=0x5AEC7000 + sd)
    T.materialize(t)
    traces.append(t)
var = A.variants()
names = list(var)
R = len(names) * a.seeds
rep_of = [sd for nm in names for sd in range(a.seeds)]
pol = C.policy_config(2304)
cache = S.SaeCache(2304, n_replicas=R, policy=pol)
for r in range(R):
    cache.set_params(r, var[names[r // a.seeds]])
batch = T.replicate(traces, rep_of)
b = S.batch_to_torch(batch)
torch.cuda.synchronize()
t0 = time.time()
out = cache.admit_batch(b)
torch.cuda.synchronize()
dt = time.time() - t0
matched = out["matched_tokens"].cpu().numpy().view(np.uint32).astype(np.int64)
L = batch["prompt_len"].astype(np.int64)
res = {"workload": a.workload, "mix": mix, "seeds": a.seeds, "requests_per_replica": a.requests,
       "replicas": R, "gpu_seconds": dt, "variants": {}}
n = a.requests
for vi, nm in enumerate(names):
    sl = slice(vi * a.seeds * n, (vi + 1) * a.seeds * n)
    pre = A.prefill_tokens(L[sl], matched[sl])
    st = [cache.stats(vi * a.seeds + s) for s in range(a.seeds)]
    hit_tok = sum(x.hit_tokens for x in st) / max(sum(x.prompt_tokens for x in st), 1)
    hit_blk = sum(x.hit_blocks for x in st) / max(sum(x.blocks_looked_up for x in st), 1)
    par = [S.params_dict(x.params) for x in st]
    res["variants"][nm] = {
        "hit_rate_tokens": hit_tok, "hit_rate_blocks": hit_blk,
        "mean_prefill_tokens": float(pre.mean()),
        "w_mean": [float(np.mean([p["w"][t] for p in par])) for t in range(5)],
        "alpha_mean": [float(np.mean([p["alpha"][q] for p in par])) for q in range(3)],
        "mu_mean": [float(np.mean([p["mu"][q] for p in par])) for q in range(2)],
        "gamma_mean": float(np.mean([p["gamma"] for p in par])),
    }
base = res["variants"]["LRU"]["mean_prefill_tokens"]
for nm, v in res["variants"].items():
    v["prefill_vs_LRU"] = v["mean_prefill_tokens"] / base
os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
json.dump(res, open(a.out + ".json", "w"), indent=1)
with open(a.out + ".md", "w") as f:
    f.write("# Baselines and ablation ladder (%s mix, %d seeds x %d requests, C = 2304)\n\n"
            % (a.workload, a.seeds, a.requests))
    f.write("| variant | token hit rate | block hit rate | mean prefill tokens | prefill vs LRU | w (sys,user,tool,resp,cot) | alpha (chat,agent,struct) |\n|---|---|---|---|---|---|---|\n")
    for nm, v in res["variants"].items():
        f.write("| %s | %.4f | %.4f | %.1f | %.3f | %s | %s |\n" % (
            nm, v["hit_rate_tokens"], v["hit_rate_blocks"], v["mean_prefill_tokens"], v["prefill_vs_LRU"],
            " ".join("%.2f" % x for x in v["w_mean"]), " ".join("%.2f" % x for x in v["alpha_mean"])))
print(open(a.out + ".md").read())
