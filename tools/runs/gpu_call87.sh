timeout 900 python -m pytest tests/test_gpu_presort.py tests/test_gpu_mcsim.py -x -q > gpurun_out/p87.log 2>&1; echo rc=$? >> gpurun_out/p87.log
timeout 900 python bench.py --no-bert --no-mcsim --no-cpu-baseline > gpurun_out/b87.json 2> gpurun_out/b87.err
B2_PRESORT_PATH=bitonic timeout 900 python bench.py --no-bert --no-mcsim --no-cpu-baseline > gpurun_out/b87b.json 2> gpurun_out/b87b.err
