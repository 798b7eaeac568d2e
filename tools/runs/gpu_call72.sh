timeout 900 python -m pytest tests/test_gpu_mcsim.py tests/test_gpu_presort.py -x -q > gpurun_out/p72.log 2>&1; echo rc=$? >> gpurun_out/p72.log
timeout 1200 python bench.py > gpurun_out/b72.json 2> gpurun_out/b72.err; echo rc=$? >> gpurun_out/b72.err
