for n in 2 4; do
for comm in fused nccl; do
for mb in 1 2 5 10 25 50 100 200; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2957$n tools/fused_bench.py --mb $mb --comm $comm --iters 10 >> gpurun_out/sweep30.jsonl 2>> gpurun_out/sweep30.err
done; done; done
