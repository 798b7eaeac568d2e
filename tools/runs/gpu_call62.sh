TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
P=29700
for c in 0 1; do P=$((P+1)); B2_FUSED_CFG=$c timeout 300 $TR --master-port $P tools/k4_timeline.py --transport nvls >> gpurun_out/t62.jsonl 2>> gpurun_out/t62.err; done
P=$((P+1)); timeout 300 $TR --master-port $P tools/k4_timeline.py --transport p2p >> gpurun_out/t62.jsonl 2>> gpurun_out/t62.err
