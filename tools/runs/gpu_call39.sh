for c in 23 27 28 29 30 31 20; do B2_CLIP_CFG=$c timeout 300 python tools/clip_bench.py --iters 30 --sweep > gpurun_out/clip39_cfg$c.jsonl 2>&1; done
