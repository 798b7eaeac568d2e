B2_FUSED_CFG=40 timeout 500 python -m pytest tests/test_gpu_multi.py -x -q -k "fused" > gpurun_out/p69.log 2>&1; echo rc=$? >> gpurun_out/p69.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
P=29700
for cs in 16 24 32 48; do P=$((P+1)); B2_COMM_SMS=$cs B2_FUSED_CFG=40 timeout 300 $TR --master-port $P tools/fused_bench.py >> gpurun_out/f69.jsonl 2>> gpurun_out/f69.err; echo "p2p cs=$cs" >> gpurun_out/f69.jsonl; done
for cs in 24 32 48 64; do P=$((P+1)); B2_COMM_SMS=$cs B2_FUSED_CFG=40 timeout 300 $TR --master-port $P tools/fused_bench.py --comm nvls >> gpurun_out/f69.jsonl 2>> gpurun_out/f69.err; echo "nvls cs=$cs" >> gpurun_out/f69.jsonl; done
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for cs in 16 24 32; do P=$((P+1)); B2_COMM_SMS=$cs B2_FUSED_CFG=40 timeout 300 $TR2 --master-port $P tools/fused_bench.py >> gpurun_out/f69.jsonl 2>> gpurun_out/f69.err; echo "n2 p2p cs=$cs" >> gpurun_out/f69.jsonl; done
