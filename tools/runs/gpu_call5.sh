timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu5.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu5.log
B2_CLIP_KERNEL=tma timeout 300 python tools/clip_bench.py --sweep > gpurun_out/clip_tma5.jsonl 2>&1
B2_CLIP_KERNEL=l2 timeout 300 python tools/clip_bench.py > gpurun_out/clip_l25.jsonl 2>&1
python tools/kernel_driver.py --only clip > gpurun_out/kd5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_bucket_clip -s 104 -c 1 -o gpurun_out/prof_tma2_batched python tools/kernel_driver.py --only clip > gpurun_out/ncu6.log 2>&1; echo ncu=$? >> gpurun_out/kd5.log
ncu --set full --clock-control none --import-source on -k regex:k_bucket_clip -s 50 -c 1 -o gpurun_out/prof_tma2_bucket python tools/kernel_driver.py --only clip > gpurun_out/ncu7.log 2>&1; echo ncu=$? >> gpurun_out/kd5.log
