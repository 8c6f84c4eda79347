"""-m gpu: the characterisation pass on the device (sae_characterize: K1 hashing + two
insert-or-find tables) equals the oracle's, counter by counter, on the hand trace and on a
30K-request balanced trace."""
import numpy as np
import pytest
import torch

import oracle
from paper_2605_18825_b200 import configs as C
from paper_2605_18825_b200 import sae as S
from paper_2605_18825_b200 import tracegen as T
from tests.test_oracle_characterize import HAND, _trace

pytestmark = pytest.mark.gpu


def _gpu(tr, single):
    cache = S.SaeCache(64, policy=C.policy_config(64))
    b = {k: tr[k] for k in ("prompt_off", "prompt_len", "decode_off", "decode_len", "tokens", "types")}
    b.update(n=tr["n"], arrival=np.arange(tr["n"], dtype=np.float64), flags=np.zeros(tr["n"], np.uint8),
             spb=np.zeros(tr["n"], np.uint32), replica=np.zeros(tr["n"], np.uint32))
    bt = S.batch_to_torch(b)
    dev = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a).astype(dt).view(
        {np.uint32: np.int32}.get(dt, dt))).cuda()
    return cache.characterize(bt, dev(tr["session"], np.uint32), dev(tr["turn"], np.uint32),
                              dev(single, np.uint8))


def test_characterize_hand_trace_gpu():
    tr = _trace(HAND)
    assert _gpu(tr, tr["single"]) == oracle.characterize(tr, C.policy_config(64), single_turn=tr["single"])


def test_characterize_balanced_trace_gpu():
    tr = T.make("c3", n_requests=30_000)
    single = (~tr["continues"]).astype(np.uint8)
    assert _gpu(tr, single) == oracle.characterize(tr, C.policy_config(64), single_turn=single)
