"""Baselines, ablation variants and the TTFT model on the same kernels.

The paper compares SAECache with LRU and LFU, and ablates it into Token-Weight-Only
and Fixed-Param Multi-Queue plus a learner ladder that adds token-weight,
log-normal, position-decay and queue-weight learning one at a time.  Each is a
parameter record (sae_params.mode / learn_flags / (mu, sigma)) for a replica of the same
sae_ctx, so a C5-style sweep replays all of them side by side on one GPU.  Prefix hits cut
the prefill work as prefill_tokens = prompt_length x (1 - hit_ratio).
"""
from __future__ import annotations

import copy

import numpy as np

from . import configs as C


def prefill_tokens(prompt_len, matched_tokens):
    """Per-request prefill tokens: prompt_length x (1 - hit_ratio) = L - matched."""
    return np.asarray(prompt_len, np.int64) - np.asarray(matched_tokens, np.int64)


def variants() -> dict:
    """name -> sae_params dict.  Fixed-Param: learners off, the chat-fitted (mu, sigma) =
    (4.15, 0.97) for both multi-turn queues.  Ladder: Fixed-Param
    + token weights, + log-normal timing, + position decay, + queue weights (= SAECache)."""
    base = copy.deepcopy(C.DEFAULT_PARAMS)
    fixed = dict(copy.deepcopy(base), learn_flags=0, mu=[4.15, 4.15], sigma=[0.97, 0.97])
    out = {
        "LRU": dict(copy.deepcopy(base), mode=C.MODE_LRU, learn_flags=0),
        "LFU": dict(copy.deepcopy(base), mode=C.MODE_LFU, learn_flags=0),
        "TokenWeightOnly": dict(copy.deepcopy(base), mode=C.MODE_TWO, learn_flags=C.L_TOKENS),
        "FixedParamMQ": fixed,
    }
    ladder = [("+token", C.L_TOKENS), ("+lognormal", C.L_TOKENS | C.L_LOGNORMAL),
              ("+decay", C.L_TOKENS | C.L_LOGNORMAL | C.L_DECAY),
              ("+queue(SAECache)", C.L_DEFAULT)]
    for name, fl in ladder:
        out["FixedParamMQ" + name] = dict(copy.deepcopy(fixed), learn_flags=fl)
    out["SAECache(relative-queue)"] = dict(copy.deepcopy(base), learn_flags=C.L_DEFAULT | C.L_QUEUE_RELATIVE)
    out["SAECache(adaptive-beta)"] = dict(copy.deepcopy(base), learn_flags=C.L_DEFAULT | C.L_ADAPTIVE_BETA)
    return out
