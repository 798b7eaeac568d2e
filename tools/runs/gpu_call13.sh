timeout 300 python -m pytest tests/test_gpu_gradsync.py -x -q > gpurun_out/pytest_gpu13.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu13.log
for c in 0 1 2 3 4 6; do B2_CLIP_CFG=$c timeout 300 python tools/clip_bench.py > gpurun_out/clip13_cfg$c.jsonl 2>&1; done
