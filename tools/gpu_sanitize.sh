#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_case.py
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
  timeout 1800 compute-sanitizer --tool $tool $extra --target-processes all --print-limit 50 \
    python tools/sanitize_case.py > gpurun_out/sanitize_${tool}.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_${tool}.log
  tail -3 gpurun_out/sanitize_${tool}.log
done
