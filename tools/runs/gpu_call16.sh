timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu16.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu16.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench16.json 2> gpurun_out/bench16.err; echo bench=$? >> gpurun_out/bench16.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench16_ref.json 2> gpurun_out/bench16_ref.err
python tools/kernel_driver.py > gpurun_out/kd16.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches16.csv python tools/kernel_driver.py > gpurun_out/ncu16a.log 2>&1; echo ncu=$? >> gpurun_out/kd16.log
ncu --set full --clock-control none --import-source on -k regex:k_bucket_clip -s 104 -c 1 -o gpurun_out/prof16_k1 python tools/kernel_driver.py --only clip > gpurun_out/ncu16b.log 2>&1; echo ncu=$? >> gpurun_out/kd16.log
