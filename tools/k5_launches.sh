# K5 per-kernel launch times (ncu gpu__time_duration, one call per case): bash tools/k5_launches.sh TAG [LIB]
TAG=$1; LIB=${2:-}
for c in in_order shuffled; do
  env ${LIB:+B2_LIB_PATH=$LIB} ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_radix --csv \
    --log-file gpurun_out/k5l_${TAG}_${c}.csv python tools/k5_bench.py --reps 1 --case $c > /dev/null 2>&1
done
