timeout 400 python -m pytest tests/test_gpu_multi.py -x -q -k fused > gpurun_out/pytest_multi24.log 2>&1; echo rc=$? >> gpurun_out/pytest_multi24.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for c in 0 2 3; do B2_FUSED_CFG=$c timeout 300 $TR --master-port 2952$c tools/fused_bench.py >> gpurun_out/fused24.jsonl 2>> gpurun_out/fused24.err; done
B2_FUSED_CFG=0 timeout 300 $TR --master-port 29530 tools/fused_bench.py --mb 100 >> gpurun_out/fused24.jsonl 2>> gpurun_out/fused24.err
