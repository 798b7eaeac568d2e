nvidia-smi topo -m > gpurun_out/topo25.txt 2>&1
timeout 500 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pytest_multi25.log 2>&1; echo rc=$? >> gpurun_out/pytest_multi25.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 4 --steps 20 --warmup 5 --no-presort > gpurun_out/bench25_n4.json 2> gpurun_out/bench25_n4.err; echo bench=$? >> gpurun_out/bench25_n4.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29542 tools/nccl_probe.py > gpurun_out/nccl25_n4.jsonl 2>&1
