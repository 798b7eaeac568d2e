#!/bin/bash
# BASELINE config 5: bucket-size sweep of the fused clip+allreduce (K4) and the NCCL step at N ranks.
# Usage (GPU box with >= N GPUs): bash tools/k4_sweep.sh N OUT.jsonl
N=$1; OUT=$2
cd "$(dirname "$0")/.."
for comm in fused nccl; do
  for mb in 1 5 10 25 50 100 200; do
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((29600 + mb)) tools/fused_bench.py --iters 20 --mb $mb --comm $comm 2>/dev/null | tail -1 >> $OUT
  done
done
