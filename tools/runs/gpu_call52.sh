TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
P=29600
for c in 11 18 19 20 21 22; do P=$((P+1)); B2_FUSED_CFG=$c timeout 300 $TR --master-port $P tools/k4_timeline.py >> gpurun_out/t52.jsonl 2>> gpurun_out/t52.err; done
for c in 18 19 20 21 22; do P=$((P+1)); B2_FUSED_CFG=$c timeout 300 $TR --master-port $P tools/fused_bench.py >> gpurun_out/f52.jsonl 2>> gpurun_out/f52.err; done
