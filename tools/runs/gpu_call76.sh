for c in 0 32 33 34 35; do B2_CLIP_CFG=$c timeout 300 python tools/clip_bench.py --iters 30 2>&1 | grep batched_bf16 | sed "s/^/c=$c /" >> gpurun_out/c76.txt; done
