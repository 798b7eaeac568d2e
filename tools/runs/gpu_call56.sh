TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
P=29800
for c in 1 0 3; do P=$((P+1)); B2_FUSED_CFG=$c timeout 300 $TR --master-port $P tools/fused_bench.py --comm nvls >> gpurun_out/f56.jsonl 2>> gpurun_out/f56.err; done
for c in 0; do P=$((P+1)); B2_FUSED_CFG=$c timeout 300 $TR --master-port $P tools/fused_bench.py --comm nvls --mb 100 >> gpurun_out/f56.jsonl 2>> gpurun_out/f56.err; done
B2_FUSED_CFG=0 timeout 400 python -m pytest tests/test_gpu_multi.py -x -q -k "nvls" > gpurun_out/p56.log 2>&1; echo rc=$? >> gpurun_out/p56.log
