"""Small fixed workload for ncu: each hot kernel a few times at BASELINE sizes.

    python tools/kernel_driver.py [--only clip|strata|presort]

Launch order (for ncu -s/-c): K1 per-bucket x 52 x 2 iters, K1 batched x 2,
K2 (3 kernels) x 2 shards, K3 lb48 epoch x 2.
"""

from __future__ import annotations

import argparse
import math
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_2402_02447_b200 as B  # noqa: E402
from paper_2402_02447_b200 import synthetic  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="all")
    ap.add_argument("--iters", type=int, default=2)
    a = ap.parse_args()
    if a.only in ("all", "clip"):
        g, layout, _ = synthetic.bert_grads(synthetic.BERT_LARGE_DIM)
        comm = torch.empty(g.numel(), dtype=torch.bfloat16, device="cuda")
        clip = B.BucketClipper()
        lim = 1.0 / math.sqrt(len(layout))
        segs = [(x, x, y - x) for x, y in reversed(layout)]
        for _ in range(a.iters):
            for s in segs:
                clip.clip_cast(g, comm, [s], lim)
        for _ in range(a.iters):
            clip.clip_cast(g, comm, segs, lim)
        torch.cuda.synchronize()
        del g, comm
    if a.only in ("all", "strata", "strata_shards", "presort"):
        lens = B.seqdata.generate_lengths(B.LengthDistribution(), 10_000_000, 2402)
        if a.only in ("all", "strata"):
            for r in range(2):
                B.stratify_lengths(lens[r * 1_250_000:(r + 1) * 1_250_000])
        if a.only in ("all", "strata_shards"):
            for _ in range(a.iters):
                B.stratify_shards(lens, [r * 1_250_000 for r in range(9)])
        if a.only in ("all", "presort"):
            n = 26_000 * 384
            ids = np.arange(n, dtype=np.int32)
            d_ids = torch.from_numpy(ids).cuda()
            d_len = torch.from_numpy(lens[:n].astype(np.int32)).cuda()
            for _ in range(a.iters):
                B.presort_deal(d_ids, d_len, 384, 8, "snake", max_len=512, max_id=n - 1)
        torch.cuda.synchronize()
    print("kernel_driver done")


if __name__ == "__main__":
    main()
