#!/bin/bash
# quick GPU pass: build, parity tests, parity report, bench, ncu of the ISM kernel
TAG=${1:-q}
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/${TAG}_pytest_gpu.log 2>&1; tail -2 gpurun_out/${TAG}_pytest_gpu.log
if [ "$2" == "parity" ]; then timeout 900 python tools/parity_report.py > gpurun_out/${TAG}_parity.txt 2>&1; cat gpurun_out/${TAG}_parity.txt; fi
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench.log 2>&1; tail -1 gpurun_out/${TAG}_bench.log | cut -c1-400
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ism_ -s 3 -c 1 -o gpurun_out/${TAG}_prof_ism python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/${TAG}_ncu.log 2>&1
tail -1 gpurun_out/${TAG}_ncu.log
