"""C4 probe: 4M-block pool, prefill then timed batches; prints select diagnostics."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_18825_b200 import configs as C, tracegen as T, sae as S
from bench import slice_batch
n_pre = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
n_step, n_steps = 2000, 5
t0 = time.time()
tr = T.make("c4", n_requests=n_pre + n_step * n_steps)
print("tracegen %.1fs tokens %d" % (time.time() - t0, tr["n_tokens"]), flush=True)
pol = C.policy_config(tr["config"]["capacity"])
cache = S.SaeCache(pol["capacity"], policy=pol)
print("GP", "created", flush=True)
t0 = time.time()
for lo in range(0, n_pre, 20000):
    b = S.batch_to_torch(slice_batch(tr, lo, min(lo + 20000, n_pre)))
    cache.admit_batch(b); torch.cuda.synchronize()
    st = cache.stats(0)
    print("prefill to %d: %.1fs resident %d evictions %d rounds %d passes %d big %d fails %s" % (
        lo + 20000, time.time() - t0, st.resident, st.evictions, st.eviction_rounds, st.select_passes,
        st.select_big, list(st.select_fail_seg)), flush=True)
s0 = cache.stats(0)
for k in range(n_steps):
    lo = n_pre + k * n_step
    b = S.batch_to_torch(slice_batch(tr, lo, lo + n_step))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); cache.admit_batch(b); e1.record(); torch.cuda.synchronize()
    st = cache.stats(0)
    print("step %d: %.1f ms -> %.0f req/s; passes %d scored %d cands/pass %.0f big %d fails %s firings %d" % (
        k, e0.elapsed_time(e1), n_step / e0.elapsed_time(e1) * 1e3, st.select_passes - s0.select_passes,
        st.blocks_scored - s0.blocks_scored,
        (st.select_cands - s0.select_cands) / max(1, st.select_passes - s0.select_passes),
        st.select_big - s0.select_big, [a - b for a, b in zip(st.select_fail_seg, s0.select_fail_seg)],
        st.learner_firings - s0.learner_firings), flush=True)
    s0 = st
print("narrows", st.select_narrow, "raw cands/pass", st.select_raw / max(1, st.select_passes))
print("resident by queue", list(st.resident_by_queue), "hit rate", st.hit_tokens / st.prompt_tokens)
print("phase ms", [round(x / 1e6, 1) for x in st.phase_ns])
