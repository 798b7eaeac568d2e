"""BERT-large samples/s under the three clip disciplines (run directly for N=1, torchrun for N>1)."""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--modes", default="stock,after,bucketwise")
    a = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if "WORLD_SIZE" in os.environ:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2402_02447_b200.train_step import bert_large_step_bench

    for m in a.modes.split(","):
        r = bert_large_step_bench(m, steps=a.steps, warmup=a.warmup)
        if int(os.environ.get("RANK", "0")) == 0:
            print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
