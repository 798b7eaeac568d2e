TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
P=29960
for w in 0 1; do for cs in 32 48 64; do P=$((P+1)); B2_K4_WIDE=$w B2_COMM_SMS=$cs timeout 300 $TR --master-port $P tools/fused_bench.py --comm nvls >> gpurun_out/f104.jsonl 2>> gpurun_out/f104.err; echo "nvls wide=$w cs=$cs" >> gpurun_out/f104.jsonl; done; done
for w in 0 1; do for cs in 48 64; do P=$((P+1)); B2_K4_WIDE=$w B2_COMM_SMS=$cs timeout 300 $TR --master-port $P tools/fused_bench.py >> gpurun_out/f104.jsonl 2>> gpurun_out/f104.err; echo "p2p wide=$w cs=$cs" >> gpurun_out/f104.jsonl; done; done
