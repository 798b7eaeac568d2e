timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu26.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu26.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench26.json 2> gpurun_out/bench26.err; echo bench=$? >> gpurun_out/bench26.err
python tools/kernel_driver.py --only presort > gpurun_out/kd26.log 2>&1 && python tools/kernel_driver.py --only strata >> gpurun_out/kd26.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches26.csv python tools/kernel_driver.py > gpurun_out/ncu26.log 2>&1; echo ncu=$? >> gpurun_out/kd26.log
