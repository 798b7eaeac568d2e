timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/p77.log 2>&1; echo rc=$? >> gpurun_out/p77.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke77.log 2>&1; echo rc=$? >> gpurun_out/smoke77.log
