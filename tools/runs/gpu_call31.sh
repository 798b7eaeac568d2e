timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu31.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu31.log
/usr/bin/time -v timeout 1200 python bench.py > gpurun_out/bench31.json 2> gpurun_out/bench31.err; echo bench=$? >> gpurun_out/bench31.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench31_ref.json 2> gpurun_out/bench31_ref.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke31.log 2>&1; echo smoke=$? >> gpurun_out/smoke31.log
