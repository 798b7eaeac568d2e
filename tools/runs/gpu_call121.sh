timeout 900 python -m pytest tests/test_gpu_multi.py -q > gpurun_out/p121.log 2>&1; echo rc=$? >> gpurun_out/p121.log
