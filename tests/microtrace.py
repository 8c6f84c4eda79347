"""Small random traces over a shared block vocabulary (prefix reuse, orphans, ghost hits,
partial blocks, decode blocks, every flag combination), for property and edge-case tests.
Input generation only: no arithmetic of the method."""
import numpy as np


def edge_trace(seed, n, one_token=False, equal_times=False, big_requests=False):
    """Small random trace over a shared block vocabulary (prefix reuse, orphans, ghosts)."""
    rng = np.random.default_rng(seed)
    vocab = [rng.integers(0, 1 << 17, 16).astype(np.uint32) for _ in range(24)]
    toks, typs, arr, po, pl, do, dl, fl, spb = [], [], [], [], [], [], [], [], []
    off, t = 0, 1.0
    for i in range(n):
        if one_token and rng.random() < 0.4:
            p = rng.integers(0, 1 << 17, 1).astype(np.uint32)
            d = np.zeros(0, np.uint32)
        else:
            nb = int(rng.integers(1, 12 if big_requests else 5))
            p = np.concatenate([vocab[int(j)] for j in rng.integers(0, len(vocab), nb)])
            p = p[: len(p) - int(rng.integers(0, 16))] if len(p) > 16 else p
            d = rng.integers(0, 1 << 17, int(rng.integers(0, 20))).astype(np.uint32)
        y = rng.integers(0, 5, len(p)).astype(np.uint8)
        po.append(off); pl.append(len(p)); toks.append(p); typs.append(y); off += len(p)
        do.append(off); dl.append(len(d)); toks.append(d); typs.append(np.full(len(d), 5, np.uint8))
        off += len(d)
        if not (equal_times and rng.random() < 0.5):
            t += float(rng.choice([1e-4, 0.5, 3.0, 40.0, 900.0]))
        arr.append(t)
        fl.append(int(rng.choice([0, 1, 3, 4, 5, 7])))
        spb.append(int(rng.integers(0, 3)))
    return {"n": n, "arrival": np.array(arr), "prompt_off": np.array(po, np.uint64),
            "prompt_len": np.array(pl, np.uint32), "decode_off": np.array(do, np.uint64),
            "decode_len": np.array(dl, np.uint32), "flags": np.array(fl, np.uint8),
            "spb": np.array(spb, np.uint32), "tokens": np.concatenate(toks),
            "types": np.concatenate(typs)}
