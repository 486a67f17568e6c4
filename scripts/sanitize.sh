#!/bin/bash
# compute-sanitizer over every kernel form (scripts/sanitize_driver.py);
# logs into gpurun_out/ (copy the summaries to profiles/).
cd "$(dirname "$0")/.."
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
  timeout 1200 $CS --tool $tool $extra --print-limit 100000 --error-exitcode 9 python scripts/sanitize_driver.py \
    > gpurun_out/r02_sanitize_$tool.log 2>&1
  echo "$tool exit $?" | tee -a gpurun_out/r02_sanitize_summary.txt
  tail -3 gpurun_out/r02_sanitize_$tool.log | tee -a gpurun_out/r02_sanitize_summary.txt
done
