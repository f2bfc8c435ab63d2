#!/bin/bash
# compute-sanitizer over tools/sanitize_case.py (run on the GPU box); logs -> gpurun_out/sanitizer_*.txt
set -u
CS=/usr/local/cuda/bin/compute-sanitizer
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check no"
  timeout 1500 $CS --tool $tool $extra --target-processes all --print-limit 50 \
      python tools/sanitize_case.py > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "$tool rc=$? $(tail -2 gpurun_out/sanitizer_$tool.txt | tr '\n' ' ')"
done
