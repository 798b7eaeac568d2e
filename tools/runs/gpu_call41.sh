for n in 2 4; do for c in 0 5 6 7; do for mb in 5 25; do
B2_FUSED_CFG=$c timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2959$n tools/fused_bench.py --mb $mb --iters 20 >> gpurun_out/fused41.jsonl 2>> gpurun_out/fused41.err
done; done; done
