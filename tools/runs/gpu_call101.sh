timeout 900 python -m pytest tests/test_gpu_multi.py -q > gpurun_out/p101.log 2>&1; echo rc=$? >> gpurun_out/p101.log
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29951 bench.py --gpus 4 > gpurun_out/b101_n4.json 2> gpurun_out/b101_n4.err
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29952 bench.py --gpus 2 > gpurun_out/b101_n2.json 2> gpurun_out/b101_n2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29953 bench.py --impl reference --gpus 2 --steps 2 --warmup 3 > gpurun_out/b101_ref_n2.json 2> gpurun_out/b101_ref_n2.err; echo rc=$? >> gpurun_out/b101_ref_n2.err
