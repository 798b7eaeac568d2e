"""Synthetic inputs of the BASELINE configs.

H1: flat fp32 gradients of BERT-base / BERT-large size in 25 MiB fp32
buckets, each bucket N(0, s_b^2) with s_b drawn (seeded) from
{1e-5, 1e-4, 1e-3} so some buckets sit below c/sqrt(B) and some above.
H2: the oracle's own Wikipedia-like generator (seqdata.generate_lengths),
sharded into contiguous rank shards, plus stratified per-step draws for a
whole epoch (the boundary input of the presort).
"""

from __future__ import annotations

import numpy as np
import torch

from .gradsync import BERT_BUCKET_ELEMS, capped_bucket_layout

BERT_BASE_DIM = 109_482_240   # 16 x 6,553,600 + 4,624,640 -> 17 buckets
BERT_LARGE_DIM = 335_141_888  # 51 x 6,553,600 + 908,288   -> 52 buckets
BUCKET_SCALES = (1e-5, 1e-4, 1e-3)


def bert_layout(dim: int) -> tuple:
    return capped_bucket_layout(dim, BERT_BUCKET_ELEMS)


def bucket_scales(num_buckets: int, seed: int = 2402) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.choice(np.asarray(BUCKET_SCALES), size=num_buckets)


def bert_grads(dim: int, seed: int = 2402, device="cuda", rank: int = 0) -> tuple:
    """(fp32 gradient vector on `device`, layout, per-bucket scales)."""
    layout = bert_layout(dim)
    scales = bucket_scales(len(layout), seed + 7919 * rank)
    gen = torch.Generator(device=device)
    gen.manual_seed(seed + rank)
    g = torch.empty(dim, dtype=torch.float32, device=device)
    for (a, b), s in zip(layout, scales):
        g[a:b].normal_(0.0, float(s), generator=gen)
    return g, layout, scales


def epoch_draws(lengths: np.ndarray, bounds, counts, num_steps: int | None, seed: int):
    """Stratified per-step draws of one rank shard for (a prefix of) an epoch.

    Returns (ids[steps, lb], lens[steps, lb]) int32: every step takes
    counts[k] samples of stratum k, without replacement across the epoch,
    stratum by stratum (the draw_batch layout, strata.py:127-141).  Steps stop
    before any stratum runs dry (no borrowing) — synthetic bench input only;
    parity tests use the host draw_batch itself.
    """
    rng = np.random.default_rng(seed)
    k_of = np.searchsorted(np.asarray(bounds), lengths, side="left")
    pools = [rng.permutation(np.flatnonzero(k_of == k)) for k in range(len(bounds))]
    steps = min((p.size // c) for p, c in zip(pools, counts) if c > 0)
    if num_steps is not None:
        steps = min(steps, num_steps)
    cols = [p[: steps * c].reshape(steps, c) for p, c in zip(pools, counts) if c > 0]
    ids = np.concatenate(cols, axis=1).astype(np.int32)
    return ids, lengths[ids].astype(np.int32)
