python bench.py --steps 10 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo bench=$? >> gpurun_out/bench1.err
python tools/kernel_driver.py > gpurun_out/kd.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/kernel_driver.py > gpurun_out/ncu1.log 2>&1; echo ncu1=$? >> gpurun_out/kd.log
ncu --set full --clock-control none --import-source on -k regex:k_bucket_clip -s 50 -c 1 -o gpurun_out/prof_clip python tools/kernel_driver.py --only clip > gpurun_out/ncu2.log 2>&1; echo ncu2=$? >> gpurun_out/kd.log
ncu --set full --clock-control none --import-source on -k regex:k_bucket_clip -s 104 -c 1 -o gpurun_out/prof_clip_batched python tools/kernel_driver.py --only clip > gpurun_out/ncu3.log 2>&1; echo ncu3=$? >> gpurun_out/kd.log
