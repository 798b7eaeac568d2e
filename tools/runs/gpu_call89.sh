timeout 900 python -m pytest tests/test_gpu_mcsim.py -x -q > gpurun_out/p89.log 2>&1; echo rc=$? >> gpurun_out/p89.log
timeout 900 python bench.py --no-bert --no-presort --no-cpu-baseline --steps 3 > gpurun_out/b89.json 2> gpurun_out/b89.err
