timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/p120.log 2>&1; echo rc=$? >> gpurun_out/p120.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke120.log 2>&1; echo rc=$? >> gpurun_out/smoke120.log
timeout 1500 python bench.py > gpurun_out/b120.json 2> gpurun_out/b120.err; echo rc=$? >> gpurun_out/b120.err
