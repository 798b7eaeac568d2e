P=29700
for c in 0 11 19; do P=$((P+1)); B2_FUSED_CFG=$c timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port $P tools/k4_timeline.py >> gpurun_out/t53.jsonl 2>> gpurun_out/t53.err; done
P=29720
for c in 19; do P=$((P+1)); B2_FUSED_CFG=$c timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P tools/k4_timeline.py --mb 100 >> gpurun_out/t53.jsonl 2>> gpurun_out/t53.err; done
