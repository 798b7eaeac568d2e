for g in 0 1 2 3 4 6; do B2_CLIP_GROUPS=$g timeout 300 python tools/clip_bench.py --iters 30 2>&1 | grep batched_bf16 | sed "s/^/g=$g /" >> gpurun_out/c75.txt; done
