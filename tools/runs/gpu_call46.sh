timeout 600 python -m pytest tests/test_gpu_presort.py -x -q -k end_to_end > gpurun_out/pytest_46a.log 2>&1; echo rc=$? >> gpurun_out/pytest_46a.log
timeout 500 python -m pytest tests/test_gpu_multi.py -x -q -k multi_bucket > gpurun_out/pytest_46b.log 2>&1; echo rc=$? >> gpurun_out/pytest_46b.log
