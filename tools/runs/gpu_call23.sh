TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for c in 0 1 2 3 4; do B2_FUSED_CFG=$c timeout 300 $TR --master-port 2952$c tools/fused_bench.py >> gpurun_out/fused23.jsonl 2>> gpurun_out/fused23.err; done
for mb in 50 100; do B2_FUSED_CFG=3 timeout 300 $TR --master-port 29530 tools/fused_bench.py --mb $mb >> gpurun_out/fused23.jsonl 2>> gpurun_out/fused23.err; done
