timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/p100.log 2>&1; echo rc=$? >> gpurun_out/p100.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke100.log 2>&1; echo rc=$? >> gpurun_out/smoke100.log
S=$(date +%s); timeout 1500 python bench.py > gpurun_out/b100.json 2> gpurun_out/b100.err; echo "rc=$? wall_s=$(( $(date +%s) - S ))" >> gpurun_out/b100.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches100.csv python bench.py --steps 2 --warmup 3 --no-bert --no-mcsim --no-cpu-baseline > gpurun_out/ncu100.log 2>&1; echo rc=$? >> gpurun_out/ncu100.log
