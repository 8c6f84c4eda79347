"""-m gpu: the hand-traced golden micro-traces (tests/golden/*.json) replayed by the CUDA
path through the C ABI (sae_admit_batch / sae_evict / sae_update / sae_stats) and checked
against the HAND-DERIVED expected values of each fixture (not against the oracle): the
same pins that fix the oracle's feedback side fix the kernels'."""
import numpy as np
import pytest
import torch

from paper_2605_18825_b200 import sae as S
from tests.golden_traces import as_trace, check_value, fixtures, policy, segments

pytestmark = pytest.mark.gpu
FIX = fixtures()


@pytest.mark.parametrize("fx", FIX, ids=[f["name"] for f in FIX])
def test_golden_trace_gpu(fx):
    pol = policy(fx)
    cache = S.SaeCache(pol["capacity"], policy=pol, traj_capacity=64)
    for kind, seg in segments(fx):
        if kind == "admit":
            tr = as_trace(seg)
            tr["replica"] = np.zeros(tr["n"], np.uint32)
            out = cache.admit_batch(S.batch_to_torch(tr))
            torch.cuda.synchronize()
            o4 = np.stack([out[k].cpu().numpy().view(np.uint32) for k in
                           ("hit_blocks", "miss_blocks", "matched_tokens", "n_victims")], 1)
            vo = out["victim_off"].cpu().numpy()
            vids = out["victim_ids"].cpu().numpy().view(np.uint32)
            for i, op in enumerate(seg):
                assert list(o4[i]) == op["out"], (fx["name"], op["t"], list(o4[i]), op["out"])
                got = [int(v) for v in vids[vo[i]:vo[i] + o4[i, 3]]]
                assert got == op["victims"], (fx["name"], op["t"], got, op["victims"])
        elif kind == "evict":
            ids, n = cache.evict(0, seg["k"], seg["t"])
            torch.cuda.synchronize()
            got = [int(v) for v in ids.cpu().numpy().view(np.uint32)[: int(n.item())]]
            assert got == seg["victims"], (fx["name"], got, seg["victims"])
        elif kind == "update":
            cache.update(0)
    st = cache.stats(0)
    for k, want in fx.get("stats", {}).items():
        got = getattr(st, k)
        check_value(k, list(got) if not isinstance(got, (int, float)) else got, want)
    par = S.params_dict(st.params)
    for k, want in fx.get("params", {}).items():
        check_value(k, par[k], want)
    if "traj" in fx:
        tj = cache.traj(0)
        assert len(tj) == len(fx["traj"])
        for a, w in zip(tj, fx["traj"]):
            assert a.E == w["E"] and a.request == w["request"]
            check_value("traj.alpha", list(a.alpha), w["alpha"])
    cache.close()
