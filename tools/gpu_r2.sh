#!/bin/bash
# round-2 GPU pass: GPU tests, cuRAND golden, bench (with sweep), optional ncu of the ISM kernel
TAG=${1:-r2}
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/${TAG}_pytest_gpu.log 2>&1; tail -3 gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python tools/gen_curand_golden.py gpurun_out/curand_philox4x32_10.txt > gpurun_out/${TAG}_curand.log 2>&1; tail -1 gpurun_out/${TAG}_curand.log
if [ "$2" != "nobench" ]; then
  timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; tail -1 gpurun_out/${TAG}_bench.log | cut -c1-600
fi
if [ "$3" == "ncu" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:ism_ -s 3 -c 1 -o gpurun_out/${TAG}_prof_ism python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-sweep --e2e-steps 2 > gpurun_out/${TAG}_ncu.log 2>&1
  tail -1 gpurun_out/${TAG}_ncu.log
fi
