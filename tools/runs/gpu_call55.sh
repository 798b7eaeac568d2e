TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
P=29800
for c in 0 10 11 12 13 14; do P=$((P+1)); B2_FUSED_CFG=$c timeout 300 $TR --master-port $P tools/fused_bench.py >> gpurun_out/f55.jsonl 2>> gpurun_out/f55.err; done
for c in 0 11 12; do P=$((P+1)); B2_FUSED_CFG=$c timeout 300 $TR --master-port $P tools/fused_bench.py --mb 100 >> gpurun_out/f55.jsonl 2>> gpurun_out/f55.err; done
P=$((P+1)); timeout 300 $TR --master-port $P tools/fused_bench.py --comm nvls >> gpurun_out/f55.jsonl 2>> gpurun_out/f55.err
