B2_K4_HYBRID=0.6 timeout 600 python -m pytest tests/test_gpu_multi.py -q -k "nvls" > gpurun_out/p113.log 2>&1; echo rc=$? >> gpurun_out/p113.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
P=29980
for h in 1.0 0.7 0.6 0.5 0.4; do for cs in 48 64; do P=$((P+1)); B2_K4_HYBRID=$h B2_COMM_SMS=$cs timeout 300 $TR --master-port $P tools/fused_bench.py --comm nvls >> gpurun_out/f113.jsonl 2>> gpurun_out/f113.err; echo "h=$h cs=$cs" >> gpurun_out/f113.jsonl; done; done
