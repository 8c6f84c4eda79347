"""Configurations C1-C5 (BASELINE.json ``configs``) and policy defaults.

Constants follow SURVEY.md §8(c) c.5 (paper values where the paper states
them, recorded readings where it is silent); DESIGN.md lists every reading.
These are *inputs* shared by the CUDA path and the oracle tests; no arithmetic
of the method lives here.
"""
from __future__ import annotations

import copy

# token types: 0 sys, 1 user, 2 tool, 3 resp, 4 cot, 5 decode
SYS, USER, TOOL, RESP, COT, DECODE = range(6)
# queues
Q_EF, Q_CHAT, Q_AGENT, Q_STRUCT = range(4)
# learner flags
L_TOKENS, L_QUEUES, L_LOGNORMAL, L_DECAY, L_TOKEN_MULT, L_QUEUE_RELATIVE = 1, 2, 4, 8, 16, 32
L_ADAPTIVE_BETA = 64   # LognormalParams' EMA factor adapts to the observation variance
L_DEFAULT = L_TOKENS | L_QUEUES | L_LOGNORMAL | L_DECAY
# eviction policy modes (include/sae.h SAE_MODE_*): the method and its baselines
MODE_SAE, MODE_LRU, MODE_LFU, MODE_TWO = 0, 1, 2, 3

HASH_SEED = 0x5AEC0000C0FFEE01

DEFAULT_PARAMS = {
    # learned values, initial (P:910-912 token weights; alpha, gamma = 1 (A: S:462);
    # (mu, sigma) chat = P:255 fixed fit, agent = CC-Bench fit P:999-1000 (A29))
    "w": [2.0, 1.5, 1.0, 1.0, 0.1],
    "alpha": [1.0, 1.0, 1.0],          # CHAT, AGENT, STRUCT
    "mu": [4.15, 2.28],                # CHAT, AGENT
    "sigma": [0.97, 1.34],
    "gamma": 1.0,
    # meta-parameters (P:703 a_miss=5, b_reuse=2; eta, T, betas chosen: A21/A22)
    "eta": 0.1, "a_miss": 5.0, "b_reuse": 2.0, "T": 2.0,
    "beta_q": 0.3, "beta_ln": 0.3, "beta_gamma": 0.3,
    "learn_flags": L_DEFAULT,
    "mode": MODE_SAE,
}


def policy_config(capacity: int, K: int = 100, ghost_capacity: int | None = None,
                  params: dict | None = None) -> dict:
    return {
        "block_tokens": 16,
        "capacity": int(capacity),
        "ghost_capacity": int(ghost_capacity if ghost_capacity is not None else capacity),  # A30
        "K": int(K),                      # chosen (P:540 silent)
        "interval_ring": 4096,            # A25
        "interval_keep": 200,
        "interval_min": 20,               # P:769 "> 20" (A23)
        "n_bins": 10,                     # A27
        "hash_seed": HASH_SEED,           # A1
        "dt_eps": 1e-3,                   # A7
        "z_cut": 30.0,                    # A36
        "params": copy.deepcopy(params or DEFAULT_PARAMS),
    }


# Table 2 category shares: chat, agent, tool_use, programming, doc_qa
MIX_MT = [0.50, 0.30, 0.10, 0.05, 0.05]
MIX_BAL = [0.30, 0.20, 0.25, 0.15, 0.10]
MIX_ST = [0.10, 0.10, 0.40, 0.25, 0.15]

CONFIGS = {
    # C1 tiny: chat 0.5 / tool_use 0.5, 4+4 templates of 48 tokens, lengths / 4
    "c1": dict(name="c1", n_requests=200, mix=[0.5, 0.0, 0.5, 0.0, 0.0], capacity=64,
               seed=0x5AEC0001, len_scale=0.25, tpl_override={"chat": (4, 48), "tool_use": (4, 48)},
               n_tpl={}, replicas=1),
    "c2": dict(name="c2", n_requests=100_000, mix=MIX_MT, capacity=2304, seed=0x5AEC0002,
               len_scale=1.0, tpl_override={}, n_tpl={}, replicas=1),
    "c3": dict(name="c3", n_requests=1_000_000, mix=MIX_BAL, capacity=16384, seed=0x5AEC0003,
               len_scale=1.0, tpl_override={}, n_tpl={}, replicas=1),
    "c4": dict(name="c4", n_requests=1_000_000, mix=MIX_ST, capacity=1 << 22, seed=0x5AEC0004,
               len_scale=1.0, tpl_override={}, n_tpl={"tool_use": 1 << 18, "programming": 1 << 16},
               replicas=1),
    # C5: 1024 replicas = 32 parameter points x 32 seeds, balanced, 10K requests, C = 2304
    "c5": dict(name="c5", n_requests=10_000, mix=MIX_BAL, capacity=2304, seed=0x5AEC1000,
               len_scale=1.0, tpl_override={}, n_tpl={}, replicas=1024),
}

# Appendix C grid: a in {0.5,1,2,5,10,20} x b in {0.5,1,2,5,10}
GRID_A = [0.5, 1.0, 2.0, 5.0, 10.0, 20.0]
GRID_B = [0.5, 1.0, 2.0, 5.0, 10.0]


def c5_point_params(point: int) -> dict:
    """Parameter point for C5 replica r (point = r mod 32): 0-29 grid, 30 learners
    off, 31 TOKEN_MULT."""
    p = copy.deepcopy(DEFAULT_PARAMS)
    if point < 30:
        p["a_miss"] = GRID_A[point // 5]
        p["b_reuse"] = GRID_B[point % 5]
    elif point == 30:
        p["learn_flags"] = 0
    else:
        p["learn_flags"] = L_DEFAULT | L_TOKEN_MULT
    return p


def get(name: str, **over) -> dict:
    c = copy.deepcopy(CONFIGS[name])
    c.update(over)
    return c
