TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
P=29700
P=$((P+1)); B2_K4_DBG=4 B2_COMM_SMS=32 B2_FUSED_CFG=40 timeout 300 $TR --master-port $P tools/k4_timeline.py --transport nvls >> gpurun_out/t68.jsonl 2>> gpurun_out/t68.err
P=$((P+1)); B2_K4_DBG=4 timeout 300 $TR --master-port $P tools/k4_timeline.py --transport p2p >> gpurun_out/t68.jsonl 2>> gpurun_out/t68.err
for c in 0 40; do P=$((P+1)); B2_K4_DBG=4 B2_COMM_SMS=24 B2_FUSED_CFG=$c timeout 300 $TR --master-port $P tools/fused_bench.py >> gpurun_out/f68.jsonl 2>> gpurun_out/f68.err; done
P=$((P+1)); B2_K4_DBG=4 B2_COMM_SMS=32 B2_FUSED_CFG=40 timeout 300 $TR --master-port $P tools/fused_bench.py --comm nvls >> gpurun_out/f68.jsonl 2>> gpurun_out/f68.err
P=$((P+1)); B2_K4_DBG=4 timeout 300 $TR --master-port $P tools/fused_bench.py --comm nvls >> gpurun_out/f68.jsonl 2>> gpurun_out/f68.err
