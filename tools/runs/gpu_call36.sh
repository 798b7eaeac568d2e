timeout 500 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pytest_multi36.log 2>&1; echo rc=$? >> gpurun_out/pytest_multi36.log
for n in 2 4; do for mb in 1 2 5 10 25 50 100 200; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2958$n tools/fused_bench.py --mb $mb --comm fused --iters 10 >> gpurun_out/sweep36.jsonl 2>> gpurun_out/sweep36.err
done; done
