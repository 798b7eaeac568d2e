timeout 300 python tools/pcie_probe.py > gpurun_out/pcie.json 2>&1
timeout 300 python tools/kernel_driver.py --only presort > gpurun_out/kd91.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_presort --launch-skip 1 --launch-count 1 -o gpurun_out/ncu_k3count python tools/kernel_driver.py --only presort > gpurun_out/ncu91.log 2>&1; echo rc=$? >> gpurun_out/ncu91.log
