timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu40.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu40.log
timeout 900 python bench.py > gpurun_out/bench40.json 2> gpurun_out/bench40.err; echo bench=$? >> gpurun_out/bench40.err
python tools/kernel_driver.py --only clip > gpurun_out/kd40.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches40.csv python tools/kernel_driver.py --only clip > gpurun_out/ncu40.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_bucket_clip_ws -s 0 -c 1 -o gpurun_out/prof40_ws python tools/kernel_driver.py --only clip > gpurun_out/ncu40b.log 2>&1; echo ncu=$? >> gpurun_out/kd40.log
