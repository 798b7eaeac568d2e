B2_K4_FORCE_R8=1 timeout 900 python -m pytest tests/test_gpu_multi.py -q -k "fused and not nvls" > gpurun_out/p114.log 2>&1; echo rc=$? >> gpurun_out/p114.log
