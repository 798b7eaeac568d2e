TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
P=29600
for c in 0 11; do for mb in 25 5; do P=$((P+1)); B2_FUSED_CFG=$c timeout 300 $TR --master-port $P tools/k4_timeline.py --mb $mb >> gpurun_out/t51.jsonl 2>> gpurun_out/t51.err; done; done
