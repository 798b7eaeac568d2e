timeout 900 python -m pytest tests/test_gpu_presort.py -x -q > gpurun_out/p88.log 2>&1; echo rc=$? >> gpurun_out/p88.log
timeout 900 python bench.py --no-bert --no-mcsim --no-cpu-baseline > gpurun_out/b88.json 2> gpurun_out/b88.err
