#!/bin/bash
# GPU tests + small-call latencies (+ their kernel durations) + optional bench
TAG=${1:-r2}
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/${TAG}_pytest_gpu.log 2>&1; tail -3 gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python tools/small_calls.py > gpurun_out/${TAG}_small.txt 2>&1; cat gpurun_out/${TAG}_small.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_small_ncu.csv python tools/small_calls.py --reps 3 > /dev/null 2>&1
if [ "$2" == "bench" ]; then
  timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; tail -1 gpurun_out/${TAG}_bench.log | cut -c1-600
fi
