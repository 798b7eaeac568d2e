nvidia-smi topo -m > gpurun_out/topo18.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pytest_multi18.log 2>&1; echo rc=$? >> gpurun_out/pytest_multi18.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench18_n2.json 2> gpurun_out/bench18_n2.err; echo bench=$? >> gpurun_out/bench18_n2.err
