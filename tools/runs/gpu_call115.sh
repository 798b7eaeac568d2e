for d in 0 1; do B2_K1_DBG=$d timeout 300 python tools/clip_bench.py --iters 30 2>&1 | grep -E "batched_bf16|norm_only" | sed "s/^/dbg=$d /" >> gpurun_out/c115.txt; done
