"""Fused clip + NVLink allreduce step (FusedBucketSync) timing, BERT-large buckets.

    B2_FUSED_CFG=k torchrun --nproc-per-node N tools/fused_bench.py [--iters 20]

Rank 0 prints one JSON line: ms per step (max over ranks, CUDA events, graph
replay) and the implied allreduce bus bandwidth of the bf16 buckets.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--mb", type=int, default=25, help="bucket size in MiB of fp32")
    ap.add_argument("--comm", choices=("fused", "nvls", "nccl"), default="fused")
    args = ap.parse_args()
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    world, rank = dist.get_world_size(), dist.get_rank()
    import paper_2402_02447_b200 as B
    from paper_2402_02447_b200 import synthetic
    from paper_2402_02447_b200.ddp import FusedBucketSync

    dim = synthetic.BERT_LARGE_DIM
    g, _, _ = synthetic.bert_grads(dim, rank=rank)
    layout = B.capped_bucket_layout(dim, args.mb * 1024 * 1024 // 4)
    if args.comm in ("fused", "nvls"):
        sync = FusedBucketSync(layout, B.ClipConfig(1.0, "bucket_wise"),
                               transport="nvls" if args.comm == "nvls" else "p2p")
        fn = lambda s_: sync.sync(g, stream=s_)  # noqa: E731
    else:
        from paper_2402_02447_b200.ddp import BucketwiseSync

        sync = BucketwiseSync(layout, B.ClipConfig(1.0, "bucket_wise"), comm_dtype=torch.bfloat16)

        def fn(s_):
            sync.sync_native(g, stream=s_)
            s_.wait_stream(sync.side)
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cap):
        fn(cap)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=cap):
        fn(cap)
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.iters):
        graph.replay()
    b.record()
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / args.iters], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    algbw = dim * 2 / (ms * 1e-3) / 1e9
    if rank == 0:
        print(json.dumps({"world": world, "comm": args.comm, "cfg": os.environ.get("B2_FUSED_CFG", "0"), "bucket_mb": args.mb,
                          "buckets": len(layout), "ms": ms, "busbw_gbs": algbw * 2 * (world - 1) / world,
                          "grad_gbs_per_rank": dim * 4 / (ms * 1e-3) / 1e9,
                          # bytes each GPU must move per direction (two-shot 2(N-1)/N of the bf16
                          # gradient, NVLS one copy) over the measured 770 GB/s peer copy
                          "nvlink_roofline_frac": (dim * 2 * (1.0 if args.comm == "nvls" else 2 * (world - 1) / world)
                                                   / 770e9 * 1e3) / ms}), flush=True)
    if hasattr(sync, "close"):
        sync.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
