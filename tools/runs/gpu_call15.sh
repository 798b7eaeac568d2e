timeout 300 python -m pytest tests/test_gpu_gradsync.py -x -q > gpurun_out/pytest_gpu15.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu15.log
for c in 6 8 9 10 11 12 13 14; do B2_CLIP_CFG=$c timeout 300 python tools/clip_bench.py > gpurun_out/clip15_cfg$c.jsonl 2>&1; done
