B2_CLIP_CFG=20 timeout 300 python -m pytest tests/test_gpu_gradsync.py -x -q > gpurun_out/pytest_gpu17.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu17.log
for c in 10 20 21 22 23 24; do B2_CLIP_CFG=$c timeout 300 python tools/clip_bench.py > gpurun_out/clip17_cfg$c.jsonl 2>&1; done
