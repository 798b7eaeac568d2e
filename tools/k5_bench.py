"""K5 alone: every 1.25M-sample rank shard of the 10M corpus sorted by (-length, id) in one call.

    python tools/k5_bench.py [--reps 10] [--case in_order|shuffled|both]

CUDA events per call (L2 flushed before each), one JSON line per case: ms, G keys/s,
GB/s at the algorithmic 12 B/key.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_2402_02447_b200 as B  # noqa: E402
from paper_2402_02447_b200.balance import presort_workspace_bytes  # noqa: E402

N, SH = 10_000_000, 8


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--case", default="both")
    a = ap.parse_args()
    shard = N // SH
    lens = B.seqdata.generate_lengths(B.LengthDistribution(), N, 2402)
    d_len = torch.from_numpy(lens.astype(np.int32)).cuda()
    rng = np.random.default_rng(5)
    cases = {}
    if a.case in ("both", "in_order"):
        cases["in_order"] = np.arange(N, dtype=np.int32)
    if a.case in ("both", "shuffled"):
        cases["shuffled"] = np.concatenate([rng.permutation(np.arange(r * shard, (r + 1) * shard, dtype=np.int32))
                                            for r in range(SH)])
    ws = torch.empty(presort_workspace_bytes(SH, shard, 512, N - 1), dtype=torch.uint8, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.float32, device="cuda")
    for name, ids in cases.items():
        d_ids = torch.from_numpy(ids).cuda()
        run = lambda: B.presort_deal(d_ids, d_len, shard, 1, "raster", max_len=512, max_id=N - 1, workspace=ws)
        for _ in range(2):
            run()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ts = []
        for _ in range(a.reps):
            flush.zero_()
            ev[0].record()
            run()
            ev[1].record()
            torch.cuda.synchronize()
            ts.append(ev[0].elapsed_time(ev[1]))
        ms = float(np.median(ts))
        print(json.dumps({"case": name, "ms": ms, "gkeys_s": N / ms / 1e6, "gbs": N * 12 / ms / 1e6}), flush=True)


if __name__ == "__main__":
    main()
