#!/bin/bash
# compute-sanitizer over every product kernel (tools/sanitize_driver.py); summaries -> gpurun_out/sanitize_*.txt
# Usage (GPU box): bash tools/sanitize.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  for part in k1 k2 k3 k5 mc k4; do
    extra=""
    [ "$tool" = "memcheck" ] && extra="--leak-check no"
    timeout 900 compute-sanitizer --tool $tool $extra --kernel-name kns=_ZN2b2 --print-limit 20 \
      python tools/sanitize_driver.py --only $part > gpurun_out/sanitize_${tool}_${part}.txt 2>&1
    echo "$tool $part rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|Error' gpurun_out/sanitize_${tool}_${part}.txt | tail -1)"
  done
done
