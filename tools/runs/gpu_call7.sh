timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu7.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu7.log
for c in 0 1 2 3 4; do B2_CLIP_CFG=$c timeout 300 python tools/clip_bench.py > gpurun_out/clip_cfg$c.jsonl 2>&1; done
B2_CLIP_CFG=1 timeout 300 python tools/clip_bench.py --sweep > gpurun_out/clip_sweep7.jsonl 2>&1
