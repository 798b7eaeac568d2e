START=$(date +%s); timeout 1200 python bench.py > gpurun_out/bench32.json 2> gpurun_out/bench32.err; echo bench=$? elapsed=$(( $(date +%s) - START ))s >> gpurun_out/bench32.err
