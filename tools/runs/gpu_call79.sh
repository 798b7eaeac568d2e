timeout 600 python -m pytest tests/test_gpu_gradsync.py -x -q > gpurun_out/p79a.log 2>&1; echo rc=$? >> gpurun_out/p79a.log
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -k "fused" > gpurun_out/p79b.log 2>&1; echo rc=$? >> gpurun_out/p79b.log
timeout 900 python bench.py --no-bert --no-presort --no-mcsim > gpurun_out/b79_n1.json 2> gpurun_out/b79_n1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29931 bench.py --gpus 2 --no-bert > gpurun_out/b79_n2.json 2> gpurun_out/b79_n2.err
