"""K3 alone: b2_presort_deal over a 10M-key epoch of node-step pools, CUDA events.

    python tools/k3_bench.py [--lb 16 48] [--reps 20]      (B2_PRESORT_PATH=bitonic|count to force a path)

Pools are 8 x lb keys of the Wikipedia-like corpus (ids random, lengths 1..512),
the bench's epoch shape; L2 flushed before every timed launch.  Prints one JSON
line per local batch: us per launch, G keys/s, HBM GB/s at 12 B/key.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_2402_02447_b200 as B  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lb", type=int, nargs="+", default=[16, 48])
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    lens = B.seqdata.generate_lengths(B.LengthDistribution(), 10_000_000, 2402)
    rng = np.random.default_rng(0)
    flush = torch.empty(256 << 20, dtype=torch.float32, device="cuda")
    for lb in a.lb:
        seg = 8 * lb
        n = (10_000_000 // seg) * seg
        ids = rng.permutation(10_000_000)[:n].astype(np.int32)
        d_ids = torch.from_numpy(ids).cuda()
        d_len = torch.from_numpy(lens[ids].astype(np.int32)).cuda()
        for _ in range(3):
            B.presort_deal(d_ids, d_len, seg, 8, "snake", max_len=512, max_id=9_999_999)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        t = []
        for _ in range(a.reps):
            flush.zero_()
            ev[0].record()
            B.presort_deal(d_ids, d_len, seg, 8, "snake", max_len=512, max_id=9_999_999)
            ev[1].record()
            torch.cuda.synchronize()
            t.append(ev[0].elapsed_time(ev[1]) * 1e3)
        us = float(np.median(t))
        print(json.dumps({"lb": lb, "keys": n, "us": us, "gkeys_s": n / us / 1e3, "gbs": n * 12 / us / 1e3,
                          "path": os.environ.get("B2_PRESORT_PATH", "default")}), flush=True)


if __name__ == "__main__":
    main()
