timeout 300 python tools/k2_driver.py > gpurun_out/k2d118.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_strata --launch-skip 4 --launch-count 2 -o gpurun_out/ncu_k2c python tools/k2_driver.py > gpurun_out/ncu118.log 2>&1; echo rc=$? >> gpurun_out/ncu118.log
