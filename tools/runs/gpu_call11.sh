timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu11.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu11.log
for m in 0 1 2; do B2_CLIP_MODE=$m timeout 300 python tools/clip_bench.py > gpurun_out/clip11_mode$m.jsonl 2>&1; done
python tools/kernel_driver.py --only clip > gpurun_out/kd11.log 2>&1 && \
B2_CLIP_MODE=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_bucket_clip -s 104 -c 1 python tools/kernel_driver.py --only clip > gpurun_out/ncu11_m1.log 2>&1; \
B2_CLIP_MODE=2 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_bucket_clip -s 104 -c 1 python tools/kernel_driver.py --only clip > gpurun_out/ncu11_m2.log 2>&1; echo ncu=$? >> gpurun_out/kd11.log
