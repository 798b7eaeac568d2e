S=$(date +%s); timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/p112.log 2>&1; echo "rc=$? wall_s=$(( $(date +%s) - S ))" >> gpurun_out/p112.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke112.log 2>&1; echo rc=$? >> gpurun_out/smoke112.log
