#!/bin/bash
# compute-sanitizer over every kernel family (tools/sanitize_cases.py), one log per tool.
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check full"
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 --error-exitcode 9 \
      python tools/sanitize_cases.py "$@" > gpurun_out/sanitize_$tool.log 2>&1
  echo "== $tool rc=$?" >> gpurun_out/sanitize_$tool.log
  tail -3 gpurun_out/sanitize_$tool.log
done
