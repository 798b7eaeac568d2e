B2_CLIP_MODE=2 timeout 120 python -m pytest tests/test_gpu_gradsync.py -x -q > gpurun_out/pytest_gpu12.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu12.log
B2_CLIP_MODE=2 timeout 300 python tools/clip_bench.py > gpurun_out/clip12_mode2.jsonl 2>&1 && \
B2_CLIP_MODE=2 python tools/kernel_driver.py --only clip > gpurun_out/kd12.log 2>&1 && \
B2_CLIP_MODE=2 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_bucket_clip -s 104 -c 1 python tools/kernel_driver.py --only clip > gpurun_out/ncu12_m2.log 2>&1; echo ncu=$? >> gpurun_out/kd12.log
