"""K2 alone: b2_strata_partition_shards over the 10M corpus (8 shards) and the 10x tiled 100M corpus.

    python tools/k2_bench.py [--reps 20]

CUDA events around each launch pair, L2 flushed before every timed run; one
JSON line per size: us, G keys/s, GB/s at the algorithmic 8 B/key.
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
from paper_2402_02447_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--sizes", type=int, nargs="+", default=[1, 10])
    a = ap.parse_args()
    lib = _lib.load()
    lens = B.seqdata.generate_lengths(B.LengthDistribution(), 10_000_000, 2402)
    flush = torch.empty(256 << 20, dtype=torch.float32, device="cuda")
    bnds = _lib.i32_array((128, 256, 384, 512))
    for reps in a.sizes:
        d = torch.from_numpy(lens).cuda().repeat(reps)
        n = d.numel()
        ws_b = lib.b2_strata_workspace_bytes(n)
        ws = torch.empty(ws_b, dtype=torch.uint8, device="cuda")
        out = torch.empty(n, dtype=torch.int32, device="cuda")
        counts = torch.empty((8, 4), dtype=torch.int64, device="cuda")
        bad = torch.empty(8, dtype=torch.int64, device="cuda")
        offs = _lib.i64_array(r * (n // 8) for r in range(9))
        sp = _lib.stream_ptr()

        def run():
            _lib.check(lib.b2_strata_partition_shards(d.data_ptr(), None, offs, 8, bnds, 4, out.data_ptr(),
                                                      counts.data_ptr(), bad.data_ptr(), ws.data_ptr(), ws_b, sp))
        for _ in range(3):
            run()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        t = []
        for _ in range(a.reps):
            flush.zero_()
            ev[0].record()
            run()
            ev[1].record()
            torch.cuda.synchronize()
            t.append(ev[0].elapsed_time(ev[1]) * 1e3)
        us = float(np.median(t))
        print(json.dumps({"keys": n, "us": us, "gkeys_s": n / us / 1e3, "gbs": n * 8 / us / 1e3}), flush=True)
        del d, ws, out


if __name__ == "__main__":
    main()
