B2_FUSED_CFG=19 timeout 300 python tools/k4_timeline.py > gpurun_out/t54.jsonl 2>&1 || exit 1
B2_FUSED_CFG=19 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_clip_allreduce --launch-skip 5 --launch-count 1 -o gpurun_out/ncu_k4_n1 python tools/k4_timeline.py > gpurun_out/ncu54.log 2>&1
echo rc=$? >> gpurun_out/ncu54.log
