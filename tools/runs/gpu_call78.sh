B2_CLIP_CFG=41 timeout 600 python -m pytest tests/test_gpu_gradsync.py -x -q > gpurun_out/p78.log 2>&1; echo rc=$? >> gpurun_out/p78.log
for c in 0 40 41 42 43 44; do B2_CLIP_CFG=$c timeout 300 python tools/clip_bench.py --iters 30 2>&1 | grep batched_bf16 | sed "s/^/c=$c /" >> gpurun_out/c78.txt; done
