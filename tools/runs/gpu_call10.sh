timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu10.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu10.log
for l in 1 2; do B2_CLIP_LAG=$l timeout 300 python tools/clip_bench.py > gpurun_out/clip10_lag$l.jsonl 2>&1; done
B2_CLIP_LAG=1 timeout 300 python tools/clip_bench.py --sweep > gpurun_out/clip10_sweep.jsonl 2>&1
python tools/kernel_driver.py --only clip > gpurun_out/kd10.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_bucket_clip -s 104 -c 1 -o gpurun_out/prof10_batched python tools/kernel_driver.py --only clip > gpurun_out/ncu10.log 2>&1; echo ncu=$? >> gpurun_out/kd10.log
