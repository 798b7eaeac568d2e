"""Per-CTA timeline of one fused K4 launch (clip + NVLink allreduce).

    B2_FUSED_CFG=k torchrun --nproc-per-node 2 tools/k4_timeline.py [--mb 25]

K4 stamps %globaltimer into spare workspace rows: 0 kernel start, 1 B (clip)
done, 2 C's first bucket ready, 3 C (reduce) done, 4 CTA exit.  Prints, per
rank, min / median / max over CTAs of each stamp in µs after the earliest
start.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

K_MAX_SEGS, K_MAX_GRID = 128, 2048
NAMES = ["start", "clip_done", "c_first_ready", "reduce_done", "exit"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=int, default=25)
    ap.add_argument("--transport", default="p2p", choices=("p2p", "nvls"))
    args = ap.parse_args()
    if "LOCAL_RANK" not in os.environ:  # single process (e.g. under ncu): a world of one
        os.environ.update(RANK="0", LOCAL_RANK="0", WORLD_SIZE="1", MASTER_ADDR="127.0.0.1", MASTER_PORT="29791")
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank = dist.get_rank()
    import paper_2402_02447_b200 as B
    from paper_2402_02447_b200 import synthetic
    from paper_2402_02447_b200.ddp import FusedBucketSync

    dim = synthetic.BERT_LARGE_DIM
    g, _, _ = synthetic.bert_grads(dim, rank=rank)
    layout = B.capped_bucket_layout(dim, args.mb * 1024 * 1024 // 4)
    sync = FusedBucketSync(layout, B.ClipConfig(1.0, "bucket_wise"), transport=args.transport)
    for _ in range(5):
        sync.sync(g)
    torch.cuda.synchronize()
    dist.barrier()
    sync.sync(g)
    torch.cuda.synchronize()
    ws = sync.clipper.workspace
    raw = ws[: K_MAX_SEGS * K_MAX_GRID * 8].view(torch.int64).view(K_MAX_SEGS, K_MAX_GRID).cpu().numpy()
    grid = torch.cuda.get_device_properties(0).multi_processor_count * 2
    st = np.stack([raw[K_MAX_SEGS - 1 - k, :grid] for k in range(5)]).astype(np.float64)
    t0 = st[0][st[0] > 0].min()
    out = {"rank": rank, "transport": args.transport, "cfg": os.environ.get("B2_FUSED_CFG", "0"), "bucket_mb": args.mb, "buckets": len(layout)}
    for k, n in enumerate(NAMES):
        v = (st[k][st[k] > 0] - t0) / 1e3  # roles stamp only their own events
        if v.size == 0:
            continue
        out[n] = [round(float(v.min()), 1), round(float(np.median(v)), 1), round(float(v.max()), 1)]
    allo = [None] * dist.get_world_size()
    dist.all_gather_object(allo, out)
    if rank == 0:
        for o in allo:
            print(json.dumps(o), flush=True)
    sync.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
