python tools/kernel_driver.py --only clip > gpurun_out/kd33.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_bucket_clip_ws -s 0 -c 1 -o gpurun_out/prof33_ws python tools/kernel_driver.py --only clip > gpurun_out/ncu33.log 2>&1; echo ncu=$? >> gpurun_out/kd33.log
