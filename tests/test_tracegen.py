"""Trace generator invariants (SURVEY §8(d) "Tracegen invariants")."""
import numpy as np

from paper_2605_18825_b200 import configs as C
from paper_2605_18825_b200 import tracegen as T


def test_splitmix_pins():
    assert T.splitmix_int(0) == 0xE220A8397B1DCDAF
    assert T.splitmix_int(1) == 0x910A2DEC89025CC1
    v = T.splitmix(np.array([0, 1, 12345], np.uint64))
    assert [int(x) for x in v] == [T.splitmix_int(0), T.splitmix_int(1), T.splitmix_int(12345)]


def small(mix, n=3000, seed=77):
    cfg = C.get("c2", n_requests=n, seed=seed, mix=mix)
    tr = T.generate(cfg)
    T.materialize(tr)
    return tr


def test_determinism_and_arrivals():
    a = small(C.MIX_BAL, 1500)
    b = small(C.MIX_BAL, 1500)
    for k in ("arrival", "prompt_off", "prompt_len", "decode_len", "flags", "spb", "tokens", "types"):
        assert np.array_equal(a[k], b[k]), k
    d = np.diff(a["arrival"])
    assert np.all(d >= 1e-6 * (1 - 1e-9))


def test_category_shares_table2():
    for mix in (C.MIX_MT, C.MIX_BAL, C.MIX_ST):
        tr = small(mix, 4000)
        got = np.bincount(tr["category"], minlength=5) / tr["n"]
        assert np.all(np.abs(got - np.asarray(mix)) <= 0.02), (got, mix)


def test_history_carry_prefix():
    """A turn-(i+1) prompt begins with the turn-i prompt plus carried output."""
    tr = small(C.MIX_MT, 3000)
    last = {}
    checked = 0
    for i in range(tr["n"]):
        s, t = int(tr["session"][i]), int(tr["turn"][i])
        po, pl = int(tr["prompt_off"][i]), int(tr["prompt_len"][i])
        p = tr["tokens"][po:po + pl]
        if (s, t - 1) in last:
            prev = last[(s, t - 1)]
            assert np.array_equal(p[: len(prev)], prev)
            checked += 1
        last[(s, t)] = p
        if t > 0:
            assert tr["flags"][i] & 4 and tr["flags"][i] & 1
    assert checked > 100


def test_templates_shared_and_content_unique():
    tr = small(C.MIX_ST, 2000)
    tool = np.nonzero(tr["category"] == 2)[0]
    first = {}
    shared = 0
    for i in tool[:300]:
        po = int(tr["prompt_off"][i])
        blk = tuple(tr["tokens"][po:po + 16])
        shared += blk in first
        first[blk] = i
    assert shared > 50     # Zipf templates repeat
    # spb = template blocks; template tokens typed sys/tool
    assert np.all(tr["spb"][tool] >= 1)
