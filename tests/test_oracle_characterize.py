"""Pin of the oracle's characterisation pass (unbounded cache, DESIGN.md
A42) on a hand-traced trace: reuse, intra- vs inter-session reuse by token type (Table 1
columns), positional bins of single-turn sessions and session locality."""
import numpy as np

import oracle
from paper_2605_18825_b200 import configs as C


def _trace(reqs):
    toks, typs, po, pl, do, dl = [], [], [], [], [], []
    off = 0
    for blocks, _, _, _ in reqs:
        t = np.concatenate([np.full(16, v, np.uint32) for v in blocks])
        po.append(off); pl.append(len(t)); toks.append(t); typs.append(np.ones(len(t), np.uint8))
        off += len(t)
        do.append(off); dl.append(0)
    return {"n": len(reqs), "prompt_off": np.array(po, np.uint64), "prompt_len": np.array(pl, np.uint32),
            "decode_off": np.array(do, np.uint64), "decode_len": np.array(dl, np.uint32),
            "tokens": np.concatenate(toks), "types": np.concatenate(typs),
            "session": np.array([r[1] for r in reqs], np.uint32), "turn": np.array([r[2] for r in reqs], np.uint32),
            "single": np.array([r[3] for r in reqs], np.uint8)}


HAND = [  # (block token values, session, turn, single-turn session)
    ([1, 2], 0, 0, 0),       # A t0: x y            nothing seen
    ([1, 2, 3], 0, 1, 0),    # A t1: x y z          x, y reused intra
    ([1, 4], 1, 0, 0),       # B t0: x w            x reused inter (seen in A)
    ([1, 4, 5], 1, 1, 0),    # B t1: x w v          x, w reused intra (B saw both at t0)
    ([1, 6], 2, 0, 1),       # C (single turn): x u  x reused inter; bins j=0 -> 0, j=1 -> 5
]


def test_characterize_hand_trace():
    tr = _trace(HAND)
    r = oracle.characterize(tr, C.policy_config(64), single_turn=tr["single"])
    assert r["blocks"] == [0, 12, 0, 0, 0, 0] and r["reused"] == [0, 6, 0, 0, 0, 0]
    assert r["later_blocks"][1] == 6 and r["later_intra"][1] == 4
    assert r["first_blocks"][1] == 6 and r["first_inter"][1] == 2
    assert r["pos_blocks"] == [1, 0, 0, 0, 0, 1, 0, 0, 0, 0]
    assert r["pos_reused"] == [1, 0, 0, 0, 0, 0, 0, 0, 0, 0]
    assert r["reuses_intra"] == 4 and r["reuses_inter"] == 2
