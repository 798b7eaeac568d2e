timeout 600 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/p71.log 2>&1; echo rc=$? >> gpurun_out/p71.log
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
TR4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
P=29700
for cs in 64 80 96; do P=$((P+1)); B2_COMM_SMS=$cs timeout 300 $TR2 --master-port $P tools/fused_bench.py >> gpurun_out/f71.jsonl 2>> gpurun_out/f71.err; echo "n2 cs=$cs" >> gpurun_out/f71.jsonl; done
for mb in 1 5 10 100 200; do P=$((P+1)); timeout 300 $TR2 --master-port $P tools/fused_bench.py --mb $mb >> gpurun_out/f71.jsonl 2>> gpurun_out/f71.err; done
for mb in 1 5 25 100; do P=$((P+1)); timeout 300 $TR4 --master-port $P tools/fused_bench.py --mb $mb >> gpurun_out/f71.jsonl 2>> gpurun_out/f71.err; done
for mb in 25 100; do P=$((P+1)); timeout 300 $TR4 --master-port $P tools/fused_bench.py --mb $mb --comm nvls >> gpurun_out/f71.jsonl 2>> gpurun_out/f71.err; done
P=$((P+1)); timeout 900 $TR4 --master-port $P bench.py --gpus 4 > gpurun_out/b71_n4.json 2> gpurun_out/b71_n4.err
P=$((P+1)); timeout 900 $TR2 --master-port $P bench.py --gpus 2 > gpurun_out/b71_n2.json 2> gpurun_out/b71_n2.err
