P=29700
for c in 0 23 24; do P=$((P+1)); B2_FUSED_CFG=$c timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port $P tools/k4_timeline.py >> gpurun_out/t58.jsonl 2>> gpurun_out/t58.err; done
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for c in 0 23 24; do P=$((P+1)); B2_FUSED_CFG=$c timeout 300 $TR --master-port $P tools/fused_bench.py >> gpurun_out/f58.jsonl 2>> gpurun_out/f58.err; done
