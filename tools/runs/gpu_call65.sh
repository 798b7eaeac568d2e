TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
B2_FUSED_CFG=40 timeout 400 python -m pytest tests/test_gpu_multi.py -x -q -k "fused and not nvls" > gpurun_out/p65.log 2>&1; echo rc=$? >> gpurun_out/p65.log
P=29700
for cs in 16 32; do P=$((P+1)); B2_COMM_SMS=$cs B2_FUSED_CFG=40 timeout 300 $TR --master-port $P tools/k4_timeline.py >> gpurun_out/t65.jsonl 2>> gpurun_out/t65.err; done
for cs in 8 16 24 32 48 64; do P=$((P+1)); B2_COMM_SMS=$cs B2_FUSED_CFG=40 timeout 300 $TR --master-port $P tools/fused_bench.py >> gpurun_out/f65.jsonl 2>> gpurun_out/f65.err; echo "cs=$cs" >> gpurun_out/f65.jsonl; done
for c in 41 42; do P=$((P+1)); B2_COMM_SMS=32 B2_FUSED_CFG=$c timeout 300 $TR --master-port $P tools/fused_bench.py >> gpurun_out/f65.jsonl 2>> gpurun_out/f65.err; done
