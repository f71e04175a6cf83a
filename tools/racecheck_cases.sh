#!/bin/bash
# racecheck per kernel case (tools/sanitize_cases.py), hazard counts per case.
#   bash tools/racecheck_cases.sh [tag]
tag=${1:-r2}
out=gpurun_out/${tag}_sanitizer
mkdir -p "$out"
: > "$out/racecheck_by_case.txt"
for c in attn_f32 attn_bf16 decode softmax quant quant_2sm rms rms_2sm layernorm routing router mla rowstats; do
  timeout 600 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 3 \
      python tools/sanitize_cases.py "$c" > "$out/racecheck_$c.txt" 2>&1
  echo "$c rc=$? $(grep -E 'RACECHECK SUMMARY|ERROR SUMMARY' "$out/racecheck_$c.txt" | tail -1)" \
      | tee -a "$out/racecheck_by_case.txt"
done
