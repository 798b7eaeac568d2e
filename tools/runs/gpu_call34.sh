timeout 900 python bench.py --steps 10 --warmup 3 --no-bert > gpurun_out/bench34.json 2> gpurun_out/bench34.err; echo bench=$? >> gpurun_out/bench34.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench34_ref.json 2> gpurun_out/bench34_ref.err; echo ref=$? >> gpurun_out/bench34_ref.err
