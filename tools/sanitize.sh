#!/bin/bash
# compute-sanitizer over tools/sanitize_run.py (run on the GPU box); logs to gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 $CS --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize_run.py \
    > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize_run' gpurun_out/sanitize_$tool.log | tr '\n' ' ')"
done
