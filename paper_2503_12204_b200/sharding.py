"""Sample sharding and the GPU-count-invariant reduction of the weighted mean.

This is the host-side statement of the multi-GPU protocol the C-ABI runs with
NCCL inside each step's CUDA graph (csrc/d4orm_cuda.cu, enqueue_step):

* rank r of G owns the contiguous samples [r·M/G, (r+1)·M/G); the Philox noise
  counter uses the *global* sample index, so the sample set is identical for
  any G;
* rewards are all-gathered, so every rank computes the same z-scored weights
  from the full vector (score_weights needs the global std — SURVEY F4);
* Σ_m w_m·sample_m is summed per chunk of CHUNK samples and the chunk partials
  are combined by a binary-counter pairwise tree (k_wmean_tree).  A rank owns an
  aligned power-of-two block of chunks, so its local root is one subtree of the
  single-GPU tree (the binary counter only merges equal-size subtrees, and a
  block of 2^k leaves closes exactly one); after all-gathering the G roots every
  rank finishes the same tree — the top of the single-GPU tree for any G — so
  the result is bitwise identical for every G whose per-rank chunk count is a
  power of two (G = 1, 2, 4, 8 at C5, and e.g. G = 3 at M = 3·2^k·256).
"""
from __future__ import annotations

import numpy as np

CHUNK = 256  # kChunk in csrc/d4orm_cuda.cu


def shard_range(M: int, world: int, rank: int) -> tuple[int, int]:
    """(first global sample, count) of `rank`."""
    if M % world:
        raise ValueError(f"batch {M} not divisible by world {world}")
    Ml = M // world
    if world > 1:
        ch = Ml // CHUNK
        if Ml % CHUNK or ch & (ch - 1):
            raise ValueError(f"per-rank batch {Ml} must be {CHUNK} x a power of two samples (world {world})")
    return rank * Ml, Ml


def pairwise_tree(parts):
    """Binary-counter pairwise sum, exactly k_wmean_tree's order: equal-size
    subtrees merge as (older + newer); leftovers fold right to left."""
    stack = []
    for cnt, v in enumerate(parts):
        k = cnt
        while k & 1:
            v = stack.pop() + v
            k >>= 1
        stack.append(v)
    total = stack.pop()
    while stack:
        total = stack.pop() + total
    return total


LARGE_E = 16384  # kPartLargeE in csrc/d4orm_cuda.cu


def chunk_partials(samples: np.ndarray, weights: np.ndarray, chunk: int = CHUNK, du: int = 2):
    """Per-chunk Σ_m w_m·sample_m in k_wmean_partial's order: each of SUB
    sub-ranges sums its LANES samples in ascending m, then the sub-sums are
    combined by a balanced pairwise tree (k5_sub in csrc/d4orm_cuda.cu: SUB = 1
    when E >= LARGE_E, 4 for the other shapes whose K5a skips zero weights —
    du = 3 — else 16)."""
    SUB = 1 if samples.shape[1] >= LARGE_E else (4 if du == 3 else 16)
    LANES = chunk // SUB
    out = []
    for c0 in range(0, samples.shape[0], chunk):
        subs = []
        for s0 in range(c0, c0 + chunk, LANES):
            acc = np.zeros(samples.shape[1:])
            for m in range(s0, min(s0 + LANES, samples.shape[0])):
                acc = acc + weights[m] * samples[m]
            subs.append(acc)
        out.append(pairwise_tree(subs))
    return out
