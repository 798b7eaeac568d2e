TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512"
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,GRAPH,TUNING timeout 300 $TR tools/nccl_probe.py > gpurun_out/nccl20_default.jsonl 2> gpurun_out/nccl20_default.err
timeout 300 $TR tools/nccl_probe.py --native > gpurun_out/nccl20_native.jsonl 2> gpurun_out/nccl20_native.err
NCCL_MIN_NCHANNELS=32 timeout 300 $TR tools/nccl_probe.py > gpurun_out/nccl20_ch32.jsonl 2> gpurun_out/nccl20_ch32.err
NCCL_NVLS_ENABLE=0 timeout 300 $TR tools/nccl_probe.py > gpurun_out/nccl20_nonvls.jsonl 2> gpurun_out/nccl20_nonvls.err
NCCL_P2P_LEVEL=NVL NCCL_ALGO=Ring timeout 300 $TR tools/nccl_probe.py > gpurun_out/nccl20_ring.jsonl 2> gpurun_out/nccl20_ring.err
