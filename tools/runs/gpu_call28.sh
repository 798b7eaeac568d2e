timeout 600 python -m pytest tests/test_gpu_presort.py -x -q > gpurun_out/pytest_gpu28.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu28.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench28.json 2> gpurun_out/bench28.err; echo bench=$? >> gpurun_out/bench28.err
