#!/bin/bash
# compute-sanitizer over tools/sanitize_cases.py: memcheck, racecheck, synccheck, initcheck; logs to gpurun_out/
cd "$(dirname "$0")/.."
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" == "racecheck" ] && extra="--racecheck-report all"
  timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool $tool $extra --print-limit 50 \
    python tools/sanitize_cases.py > gpurun_out/sanitize_${tool}.log 2>&1
  echo "$tool rc=$? $(grep -c '^ok' gpurun_out/sanitize_${tool}.log) cases; $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_${tool}.log | tail -1)"
done
