for c in 0 5 10; do B2_CLIP_CFG=$c timeout 300 python tools/clip_bench.py --iters 30 2>&1 | grep -E "single_25MiB|per_bucket_bf16_graph" | sed "s/^/c=$c /" >> gpurun_out/c97.txt; done
