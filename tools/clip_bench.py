"""K1 micro-benchmark: per-bucket vs batched launches, out dtypes, bucket-size sweep.

    B2_CLIP_KERNEL=tma|l2 python tools/clip_bench.py [--iters 20]

Prints one JSON object per configuration (CUDA-event timing, inputs 1.34 GB >
L2 so every iteration streams from HBM).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_2402_02447_b200 as B  # noqa: E402
from paper_2402_02447_b200 import synthetic  # noqa: E402

HBM = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
    if (Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").exists() else 6650.0


def timed(fn, iters):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters * 1e-3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--sweep", action="store_true")
    args = ap.parse_args()
    variant = os.environ.get("B2_CLIP_KERNEL", "tma")
    dim = synthetic.BERT_LARGE_DIM
    g, layout, _ = synthetic.bert_grads(dim)
    clip = B.BucketClipper()
    lim = 1.0 / math.sqrt(len(layout))
    segs = [(a, a, b - a) for a, b in reversed(layout)]
    out16 = torch.empty(dim, dtype=torch.bfloat16, device="cuda")
    out32 = torch.empty(dim, dtype=torch.float32, device="cuda")

    def rep(name, secs, bytes_):
        gbs = bytes_ / secs / 1e9
        print(json.dumps({"variant": variant, "case": name, "us": secs * 1e6, "gbs": gbs, "frac": gbs / HBM}), flush=True)

    rep("per_bucket_bf16_unprepared", timed(lambda: [clip.clip_cast(g, out16, [s], lim) for s in segs], args.iters), dim * 6)
    launchers = [clip.prepare(g, out16, [s], lim) for s in segs]
    rep("per_bucket_bf16", timed(lambda: [f() for f in launchers], args.iters), dim * 6)
    # the same 52 launches captured once into a CUDA graph (no host launch cost)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        gclip = B.BucketClipper(stream=side)
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=side):
            gl = [gclip.prepare(g, out16, [s], lim) for s in segs]
            for f in gl:
                f()
    torch.cuda.synchronize()
    rep("per_bucket_bf16_graph", timed(graph.replay, args.iters), dim * 6)
    rep("batched_bf16", timed(lambda: clip.clip_cast(g, out16, segs, lim), args.iters), dim * 6)
    rep("batched_f32", timed(lambda: clip.clip_cast(g, out32, segs, lim), args.iters), dim * 8)
    norms = torch.empty(len(segs), dtype=torch.float64, device="cuda")
    rep("norm_only", timed(lambda: clip.clip_cast(g, None, segs, lim, norms=norms), args.iters), dim * 4)
    one = segs[1]
    f1 = clip.prepare(g, out16, [one], lim)
    rep("single_25MiB_bucket_bf16", timed(f1, args.iters * 10), one[2] * 6)
    if args.sweep:
        for mb in (1, 2, 5, 10, 25, 50, 100, 200):
            n = mb * 1024 * 1024 // 4
            lay = B.capped_bucket_layout(dim, n)
            ss = [(a, a, b - a) for a, b in reversed(lay)]
            lim2 = 1.0 / math.sqrt(len(lay))
            rep(f"sweep_batched_{mb}MB", timed(lambda: clip.clip_cast(g, out16, ss, lim2), args.iters), dim * 6)
            rep(f"sweep_per_bucket_{mb}MB", timed(lambda: [clip.clip_cast(g, out16, [s], lim2) for s in ss], max(3, args.iters // 4)), dim * 6)


if __name__ == "__main__":
    main()
