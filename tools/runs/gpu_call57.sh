timeout 600 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/p57.log 2>&1; echo rc=$? >> gpurun_out/p57.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29811 bench.py --gpus 4 > gpurun_out/b57_n4.json 2> gpurun_out/b57_n4.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29812 bench.py --gpus 2 > gpurun_out/b57_n2.json 2> gpurun_out/b57_n2.err
