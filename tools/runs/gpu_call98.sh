timeout 900 python -m pytest tests/test_gpu_presort.py tests/test_gpu_mcsim.py -x -q > gpurun_out/p98.log 2>&1; echo rc=$? >> gpurun_out/p98.log
timeout 900 python bench.py --no-bert --no-mcsim --no-cpu-baseline > gpurun_out/b98.json 2> gpurun_out/b98.err
