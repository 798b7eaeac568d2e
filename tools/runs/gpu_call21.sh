timeout 400 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pytest_multi21.log 2>&1; echo rc=$? >> gpurun_out/pytest_multi21.log
