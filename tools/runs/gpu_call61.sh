TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
P=29700
for c in 0 30 31 34; do P=$((P+1)); B2_FUSED_CFG=$c timeout 300 $TR --master-port $P tools/k4_timeline.py >> gpurun_out/t61.jsonl 2>> gpurun_out/t61.err; done
