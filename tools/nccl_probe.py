"""NCCL allreduce bus-bandwidth probe (torchrun, one rank per GPU).

    torchrun --nproc-per-node N tools/nccl_probe.py [--native]

Prints one JSON line per message size (bf16, in place, avg) from rank 0:
algbw = bytes / time, busbw = algbw * 2 (n-1) / n.
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
    ap.add_argument("--native", action="store_true", help="use libb2ddp's NCCL communicator")
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    world, rank = dist.get_world_size(), dist.get_rank()
    comm = None
    if args.native:
        from paper_2402_02447_b200.ddp import NcclComm

        comm = NcclComm()
    for mb in (1, 4, 13, 26, 64, 256, 670):
        n = mb * 1024 * 1024 // 2
        x = torch.ones(n, dtype=torch.bfloat16, device="cuda")
        ar = (lambda: comm.all_reduce_avg(x)) if comm else (lambda: dist.all_reduce(x, op=dist.ReduceOp.AVG))
        for _ in range(5):
            ar()
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.iters):
            ar()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / args.iters
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        algbw = n * 2 / (ms * 1e-3) / 1e9
        if rank == 0:
            print(json.dumps({"world": world, "MB": mb, "us": ms * 1e3, "algbw_gbs": algbw,
                              "busbw_gbs": algbw * 2 * (world - 1) / world, "native": args.native,
                              "env": {k: v for k, v in os.environ.items() if k.startswith("NCCL_")}}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
