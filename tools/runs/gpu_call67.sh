TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
P=29700
for cs in 24 40 56; do P=$((P+1)); B2_COMM_SMS=$cs B2_FUSED_CFG=40 timeout 300 $TR --master-port $P tools/fused_bench.py >> gpurun_out/f67.jsonl 2>> gpurun_out/f67.err; echo "p2p cs=$cs" >> gpurun_out/f67.jsonl; done
for cs in 16 32 48; do P=$((P+1)); B2_COMM_SMS=$cs B2_FUSED_CFG=40 timeout 300 $TR --master-port $P tools/fused_bench.py --comm nvls >> gpurun_out/f67.jsonl 2>> gpurun_out/f67.err; echo "nvls cs=$cs" >> gpurun_out/f67.jsonl; done
P=$((P+1)); B2_COMM_SMS=32 B2_FUSED_CFG=40 timeout 300 $TR --master-port $P tools/k4_timeline.py --transport nvls >> gpurun_out/t67.jsonl 2>> gpurun_out/t67.err
