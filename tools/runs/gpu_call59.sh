P=29700
for c in 30 33; do P=$((P+1)); B2_FUSED_CFG=$c timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port $P tools/k4_timeline.py >> gpurun_out/t59.jsonl 2>> gpurun_out/t59.err; done
B2_FUSED_CFG=30 timeout 400 python -m pytest tests/test_gpu_multi.py -x -q -k "fused and not nvls" > gpurun_out/p59.log 2>&1; echo rc=$? >> gpurun_out/p59.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for c in 0 30 31 32 33 34; do P=$((P+1)); B2_FUSED_CFG=$c timeout 300 $TR --master-port $P tools/fused_bench.py >> gpurun_out/f59.jsonl 2>> gpurun_out/f59.err; done
for c in 0 31 33; do P=$((P+1)); B2_FUSED_CFG=$c timeout 300 $TR --master-port $P tools/fused_bench.py --mb 5 >> gpurun_out/f59.jsonl 2>> gpurun_out/f59.err; done
