timeout 600 python -m pytest tests/test_gpu_gradsync.py -x -q > gpurun_out/pytest_gpu35.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu35.log
timeout 600 python tools/clip_bench.py --sweep > gpurun_out/clip35.jsonl 2>&1
