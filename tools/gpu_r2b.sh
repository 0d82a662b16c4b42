#!/bin/bash
# round-2 GPU pass: GPU tests, bench (default line with sweep), ncu launch list, ncu --set full of the ISM kernel
TAG=${1:-r2}
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -2 gpurun_out/${TAG}_smoke.log
timeout 1500 python -m pytest tests -q -m gpu ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/${TAG}_pytest_gpu.log 2>&1; tail -3 gpurun_out/${TAG}_pytest_gpu.log
if [ "$2" != "nobench" ]; then
  timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; tail -1 gpurun_out/${TAG}_bench.log | cut -c1-400
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sweep --e2e-steps 1 > /dev/null 2>&1
fi
if [ "$3" == "ncu" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:ism_ -s 3 -c 1 -o gpurun_out/${TAG}_prof_ism python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-sweep --e2e-steps 1 > gpurun_out/${TAG}_ncu.log 2>&1
  tail -1 gpurun_out/${TAG}_ncu.log
fi
