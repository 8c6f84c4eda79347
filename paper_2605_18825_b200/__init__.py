"""SAECache hot path on B200 (arxiv 2605.18825): batched trace replay of the
semantic-adaptive prefix-cache eviction policy, as hand-written sm_100a CUDA
behind the C ABI in include/sae.h.

Importing the package does not load the CUDA library; ``paper_2605_18825_b200.sae``
does, and fails loudly if it is missing (there is no CPU fallback).
"""
__all__ = ["configs", "tracegen"]
