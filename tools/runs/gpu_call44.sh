timeout 300 python -m pytest tests/test_gpu_multi.py -x -q -k "nvls or fused" > gpurun_out/pytest_multi44.log 2>&1; echo rc=$? >> gpurun_out/pytest_multi44.log
for n in 2 4; do for comm in nvls fused; do for mb in 5 25 100; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2961$n tools/fused_bench.py --mb $mb --comm $comm --iters 20 >> gpurun_out/fused44.jsonl 2>> gpurun_out/fused44.err
done; done; done
