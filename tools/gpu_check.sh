#!/bin/bash
# Standard GPU pass (run under gpurun): build, smoke, parity tests, bench, launch list, ncu of the ISM kernel.
# usage: tools/gpu_check.sh [tag] [skip_tests]
TAG=${1:-run}
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1 || { tail -20 gpurun_out/${TAG}_smoke.log; }
if [ "$2" != "skip_tests" ]; then
  timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/${TAG}_pytest_gpu.log 2>&1
  tail -5 gpurun_out/${TAG}_pytest_gpu.log
fi
timeout 600 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; tail -1 gpurun_out/${TAG}_bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ism_ -s 3 -c 1 \
   -o gpurun_out/${TAG}_prof_ism python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/${TAG}_ncu.log 2>&1
tail -3 gpurun_out/${TAG}_ncu.log
