TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
P=29600
for c in 11 14 15 16 17 0; do P=$((P+1)); B2_FUSED_CFG=$c timeout 300 $TR --master-port $P tools/fused_bench.py >> gpurun_out/f50.jsonl 2>> gpurun_out/f50.err; done
for mb in 5 100; do for c in 11 14 15; do P=$((P+1)); B2_FUSED_CFG=$c timeout 300 $TR --master-port $P tools/fused_bench.py --mb $mb >> gpurun_out/f50.jsonl 2>> gpurun_out/f50.err; done; done
B2_FUSED_CFG=15 timeout 400 python -m pytest tests/test_gpu_multi.py -x -q -k "fused and not nvls" > gpurun_out/p50.log 2>&1; echo rc=$? >> gpurun_out/p50.log
