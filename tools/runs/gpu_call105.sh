timeout 900 python -m pytest tests/test_gpu_multi.py -q -k fused > gpurun_out/p105.log 2>&1; echo rc=$? >> gpurun_out/p105.log
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29971 bench.py --gpus 4 --no-bert --no-presort --no-mcsim > gpurun_out/b105_n4.json 2> gpurun_out/b105_n4.err
