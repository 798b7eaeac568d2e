TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
P=29700
for cs in 40 56 64 80; do P=$((P+1)); B2_COMM_SMS=$cs B2_FUSED_CFG=40 timeout 300 $TR --master-port $P tools/fused_bench.py >> gpurun_out/f70.jsonl 2>> gpurun_out/f70.err; echo "n4 p2p cs=$cs" >> gpurun_out/f70.jsonl; done
for cs in 48 64; do P=$((P+1)); B2_COMM_SMS=$cs B2_FUSED_CFG=41 timeout 300 $TR --master-port $P tools/fused_bench.py >> gpurun_out/f70.jsonl 2>> gpurun_out/f70.err; echo "n4 p2p cfg41 cs=$cs" >> gpurun_out/f70.jsonl; done
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for cs in 40 48 64; do P=$((P+1)); B2_COMM_SMS=$cs B2_FUSED_CFG=40 timeout 300 $TR2 --master-port $P tools/fused_bench.py >> gpurun_out/f70.jsonl 2>> gpurun_out/f70.err; echo "n2 p2p cs=$cs" >> gpurun_out/f70.jsonl; done
for c in 41 42; do P=$((P+1)); B2_COMM_SMS=40 B2_FUSED_CFG=$c timeout 300 $TR2 --master-port $P tools/fused_bench.py >> gpurun_out/f70.jsonl 2>> gpurun_out/f70.err; echo "n2 cfg$c cs=40" >> gpurun_out/f70.jsonl; done
for mb in 5 100; do P=$((P+1)); B2_COMM_SMS=40 B2_FUSED_CFG=40 timeout 300 $TR2 --master-port $P tools/fused_bench.py --mb $mb >> gpurun_out/f70.jsonl 2>> gpurun_out/f70.err; echo "n2 cs=40 mb=$mb" >> gpurun_out/f70.jsonl; done
