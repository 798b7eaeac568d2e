TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
P=29700
for d in 2 1; do for t in nvls p2p; do P=$((P+1)); B2_K4_DBG=$d timeout 300 $TR --master-port $P tools/k4_timeline.py --transport $t >> gpurun_out/t63.jsonl 2>> gpurun_out/t63.err; done; done
