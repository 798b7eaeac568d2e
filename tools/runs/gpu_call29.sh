timeout 600 python tools/bert_bench.py --steps 10 --warmup 3 > gpurun_out/bert29_n1.jsonl 2> gpurun_out/bert29_n1.err; echo rc=$? >> gpurun_out/bert29_n1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 tools/bert_bench.py --steps 10 --warmup 3 > gpurun_out/bert29_n2.jsonl 2> gpurun_out/bert29_n2.err; echo rc=$? >> gpurun_out/bert29_n2.err
timeout 400 python -m pytest tests/test_gpu_multi.py -x -q -k presort > gpurun_out/pytest_multi29.log 2>&1; echo rc=$? >> gpurun_out/pytest_multi29.log
