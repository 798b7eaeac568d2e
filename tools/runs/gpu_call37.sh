timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu37.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu37.log
timeout 900 python bench.py --steps 2 --warmup 1 --no-bert --no-cpu-baseline > gpurun_out/bench37_plain.json 2> gpurun_out/bench37_plain.err && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file gpurun_out/bench37_launches.csv python bench.py --steps 2 --warmup 1 --no-bert --no-cpu-baseline > gpurun_out/ncu37.log 2>&1; echo ncu=$? >> gpurun_out/bench37_plain.err
