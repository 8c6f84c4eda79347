"""-m gpu parity of the tensor-core session predictor (csrc/predictor.cu, Eq.(4))
with the fp64 oracle (oracle/predictor.py): every logit within the bound derived from the
kernel's arithmetic (tests/predictor_bound.py), every prediction equal where the oracle's
|y| exceeds that bound (elsewhere either answer is a correct rounding).  Ragged batches
(1, 255, 256, 257, 1000 rows: partial 128-row M tiles and 256-row CTA tiles), the paper-scale
d = 4096, the serving model's d = 1536 and the minimum d = 32, the bench's full size
(sampled rows), the flags/rows output path."""
import numpy as np
import pytest
import torch

from oracle import predictor as OP
from paper_2605_18825_b200 import predgen as PG
from paper_2605_18825_b200 import sae as S
from tests.predictor_bound import error_bound

pytestmark = pytest.mark.gpu

_W = {}


def weights(d):
    if d not in _W:
        _W[d] = PG.weights(d)
    return _W[d]


def check(h, W, y_gpu, rows=None):
    y_ref, p_ref = OP.predict(h, W)
    bound = error_bound(h, W)
    err = np.abs(y_gpu.astype(np.float64) - y_ref)
    bad = np.nonzero(err > bound)[0]
    assert bad.size == 0, ("rows outside the bound", bad[:10], err[bad[:10]], bound[bad[:10]])
    sure = np.abs(y_ref) > bound
    assert np.array_equal((y_gpu > 0)[sure], p_ref[sure])
    return err, bound


@pytest.mark.parametrize("n", [1, 255, 256, 257, 1000])
def test_predictor_ragged_batches(n):
    d = 4096
    W = weights(d)
    h = PG.hidden(n, d, seed=100 + n)
    P = S.SessionPredictor(W["w1"], W["b1"], W["w2"], W["b2"], W["w3"], W["b3"])
    y = P.predict(torch.from_numpy(h.view(np.int16)).cuda()).cpu().numpy()
    err, bound = check(h, W, y)
    # the bound is worst-case; the kernel is far inside it (a layout slip is not)
    assert np.median(err / bound) < 0.05
    assert P.launches() == 1


@pytest.mark.parametrize("d", [32, 1536])
def test_predictor_other_widths(d):
    W = weights(d)
    h = PG.hidden(700, d, seed=d)
    P = S.SessionPredictor(W["w1"], W["b1"], W["w2"], W["b2"], W["w3"], W["b3"])
    y = P.predict(torch.from_numpy(h.view(np.int16)).cuda()).cpu().numpy()
    check(h, W, y)


def test_predictor_full_size_sampled():
    # bench.py's predictor workload: 2^17 hidden states of d = 4096 (1 GiB); 4096 sampled rows
    d, n = 4096, 1 << 17
    W = weights(d)
    h = PG.hidden(n, d, seed=0x5AEC2001)
    P = S.SessionPredictor(W["w1"], W["b1"], W["w2"], W["b2"], W["w3"], W["b3"])
    y = P.predict(torch.from_numpy(h.view(np.int16)).cuda()).cpu().numpy()
    idx = np.sort(np.random.default_rng(5).choice(n, 4096, replace=False))
    idx = np.concatenate([idx, [0, 255, 256, n - 1]])
    check(h[idx], W, y[idx])
    assert np.isfinite(y).all()


def test_predictor_flags_and_rows():
    d, n = 4096, 600
    W = weights(d)
    h = PG.hidden(n, d, seed=9)
    rng = np.random.default_rng(1)
    rows = rng.permutation(n + 50)[:n].astype(np.int32)
    flags0 = rng.integers(0, 256, n + 50).astype(np.uint8)
    P = S.SessionPredictor(W["w1"], W["b1"], W["w2"], W["b2"], W["w3"], W["b3"])
    flags = torch.from_numpy(flags0.copy()).cuda()
    logit = torch.full((n + 50,), np.nan, dtype=torch.float32, device="cuda")
    P.predict(torch.from_numpy(h.view(np.int16)).cuda(), rows=torch.from_numpy(rows).cuda(), logit=logit,
              flags=flags)
    f, lg = flags.cpu().numpy(), logit.cpu().numpy()
    untouched = np.setdiff1d(np.arange(n + 50), rows)
    assert np.array_equal(f[untouched], flags0[untouched]) and np.isnan(lg[untouched]).all()
    assert np.array_equal(f[rows] & 0xFE, flags0[rows] & 0xFE)
    assert np.array_equal(f[rows] & 1, (lg[rows] > 0).astype(np.uint8))
    check(h, W, lg[rows])


def test_predictor_empty_batch_and_errors():
    W = weights(4096)
    P = S.SessionPredictor(W["w1"], W["b1"], W["w2"], W["b2"], W["w3"], W["b3"])
    out = torch.zeros(0, dtype=torch.float32, device="cuda")
    P.predict(torch.zeros((0, 4096), dtype=torch.int16, device="cuda"), logit=out)
    assert P.launches() == 0
    with pytest.raises(S.SaeError):
        S.SessionPredictor(W["w1"][:, :40], W["b1"], W["w2"], W["b2"], W["w3"], W["b3"])
