python tools/kernel_driver.py --only strata_shards > gpurun_out/kd27.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_strata -s 2 -c 2 -o gpurun_out/prof27_strata python tools/kernel_driver.py --only strata_shards > gpurun_out/ncu27.log 2>&1; echo ncu=$? >> gpurun_out/kd27.log
python tools/kernel_driver.py --only presort > gpurun_out/kd27b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_presort -s 1 -c 1 -o gpurun_out/prof27_presort python tools/kernel_driver.py --only presort > gpurun_out/ncu27b.log 2>&1; echo ncu=$? >> gpurun_out/kd27b.log
