timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu8.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu8.log
for c in 0 1 2; do B2_CLIP_CFG=$c timeout 300 python tools/clip_bench.py > gpurun_out/clip8_cfg$c.jsonl 2>&1; done
python tools/kernel_driver.py --only clip > gpurun_out/kd8.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_bucket_clip -s 104 -c 1 -o gpurun_out/prof8_batched python tools/kernel_driver.py --only clip > gpurun_out/ncu8.log 2>&1; echo ncu=$? >> gpurun_out/kd8.log
