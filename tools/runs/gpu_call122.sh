for r in 1 2 3; do timeout 300 python tools/clip_bench.py --iters 30 2>&1 | grep -E "batched_bf16" | sed "s/^/r=$r /" >> gpurun_out/c122.txt; done
