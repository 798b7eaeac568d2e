TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
P=29600
for c in 0 10 11 12 13; do P=$((P+1)); B2_FUSED_CFG=$c timeout 300 $TR --master-port $P tools/fused_bench.py >> gpurun_out/f49.jsonl 2>> gpurun_out/f49.err; done
for mb in 5 100; do for c in 0 10; do P=$((P+1)); B2_FUSED_CFG=$c timeout 300 $TR --master-port $P tools/fused_bench.py --mb $mb >> gpurun_out/f49.jsonl 2>> gpurun_out/f49.err; done; done
