timeout 300 python tools/mc_driver.py > gpurun_out/mcd.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mc --launch-skip 2 --launch-count 2 -o gpurun_out/ncu_mc python tools/mc_driver.py > gpurun_out/ncu124.log 2>&1; echo rc=$? >> gpurun_out/ncu124.log
