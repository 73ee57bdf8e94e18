#!/usr/bin/env bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over
# tools/sanitize_workload.py (run on the GPU box; logs under gpurun_out/).
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check full"
  timeout 1200 $CS --tool $tool $extra --print-limit 50 --error-exitcode 9 python tools/sanitize_workload.py \
    > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitizer_summary.txt
done
