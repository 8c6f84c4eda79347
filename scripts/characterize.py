"""Characterisation pass on the GPU: the synthetic workloads' reuse
structure with an unbounded cache -- Table 1's intra / inter / combined reuse by token type
(P:217-232), positional reuse of single-turn prompts (Fig. 2c) and session locality
 -- to compare with the paper's shape.  Writes <out>.json / .md."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2605_18825_b200 import configs as C
from paper_2605_18825_b200 import sae as S
from paper_2605_18825_b200 import tracegen as T

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/characterize"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200_000
names = ["system", "user", "tool", "response", "cot", "decode"]
res = {}
cache = S.SaeCache(64, policy=C.policy_config(64))
for wl, mix in (("multi_turn_dominant", C.MIX_MT), ("balanced", C.MIX_BAL), ("single_turn_dominant", C.MIX_ST)):
    tr = T.make("c3", n_requests=n, mix=mix)
    b = {k: tr[k] for k in ("prompt_off", "prompt_len", "decode_off", "decode_len", "tokens", "types",
                            "arrival", "flags", "spb")}
    b.update(n=tr["n"], replica=np.zeros(tr["n"], np.uint32))
    bt = S.batch_to_torch(b)
    dev = lambda a, dt, tv: torch.from_numpy(np.ascontiguousarray(a).astype(dt).view(tv)).cuda()
    torch.cuda.synchronize()
    t0 = time.time()
    r = cache.characterize(bt, dev(tr["session"], np.uint32, np.int32), dev(tr["turn"], np.uint32, np.int32),
                           dev(~tr["continues"], np.uint8, np.uint8))
    dt = time.time() - t0
    f = lambda a, b_: a / b_ if b_ else None
    res[wl] = {"requests": n, "blocks": int(bt["total_blocks"]), "seconds": dt,
               "by_type": {names[t]: {"intra_conv": f(r["later_intra"][t], r["later_blocks"][t]),
                                      "inter_conv": f(r["first_inter"][t], r["first_blocks"][t]),
                                      "combined": f(r["reused"][t], r["blocks"][t])} for t in range(6)},
               "positional_reuse_single_turn": [f(a, b_) for a, b_ in zip(r["pos_reused"], r["pos_blocks"])],
               "intra_session_share_of_reuses": f(r["reuses_intra"], r["reuses_intra"] + r["reuses_inter"]),
               "raw": r}
json.dump(res, open(out + ".json", "w"), indent=1)
with open(out + ".md", "w") as fh:
    fh.write("# Characterisation pass (unbounded cache, %d requests per mix, GPU)\n\n" % n)
    fh.write("Paper's Table 1 (real traces, P:221-231) for context: system 96.0/85.7/92.3, user 43.3/13.6/30.8, "
             "response 36.3/1.5/27.8, tool 31.2/12.2/23.0, CoT 4.2/0.0/2.2 (intra/inter/combined %).\n\n")
    for wl, v in res.items():
        fh.write("## %s (%d blocks, %.2f s on the GPU)\n\n| type | intra-conv. %% | inter-conv. %% | combined %% |\n|---|---|---|---|\n"
                 % (wl, v["blocks"], v["seconds"]))
        for nm, x in v["by_type"].items():
            p = lambda y: "-" if y is None else "%.1f" % (100 * y)
            fh.write("| %s | %s | %s | %s |\n" % (nm, p(x["intra_conv"]), p(x["inter_conv"]), p(x["combined"])))
        fh.write("\npositional reuse of single-turn prompt blocks by decile: %s\n\nintra-session share of all reuses: %.3f\n\n"
                 % (" ".join("-" if y is None else "%.2f" % y for y in v["positional_reuse_single_turn"]),
                    v["intra_session_share_of_reuses"]))
print(open(out + ".md").read())
