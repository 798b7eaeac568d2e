for c in 6 7 8 9 10; do B2_CLIP_CFG=$c timeout 300 python tools/clip_bench.py > gpurun_out/clip14_cfg$c.jsonl 2>&1; done
B2_CLIP_CFG=6 python tools/kernel_driver.py --only clip > gpurun_out/kd14.log 2>&1 && \
B2_CLIP_CFG=6 ncu --set full --clock-control none --import-source on -k regex:k_bucket_clip -s 104 -c 1 -o gpurun_out/prof14_cfg6 python tools/kernel_driver.py --only clip > gpurun_out/ncu14.log 2>&1; echo ncu=$? >> gpurun_out/kd14.log
