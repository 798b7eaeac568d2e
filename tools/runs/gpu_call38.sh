timeout 300 python -m pytest tests/test_gpu_gradsync.py -x -q > gpurun_out/pytest_gpu38.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu38.log
for c in 20 21 22 23 25 26; do B2_CLIP_CFG=$c timeout 300 python tools/clip_bench.py --iters 30 > gpurun_out/clip38_cfg$c.jsonl 2>&1; done
