#!/bin/bash
# compute-sanitizer over the smallest parity shape of every librf_cuda kernel
# (tools/sanitize_cases.py), one tool at a time; summaries into gpurun_out/.
#   bash tools/sanitize_all.sh [tag]
tag=${1:-r2}
out=gpurun_out/${tag}_sanitizer
mkdir -p "$out"
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
  timeout 1200 compute-sanitizer --tool "$tool" $extra --error-exitcode 17 \
      python tools/sanitize_cases.py > "$out/$tool.txt" 2>&1
  echo "$tool rc=$?" | tee -a "$out/summary.txt"
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|case " "$out/$tool.txt" | tee -a "$out/summary.txt"
done
