#!/bin/bash
# GPU pass without the test suite: build, bench (with the in-run parity / oracle leg), ncu --set full of the ISM kernel
TAG=${1:-b}
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; tail -1 gpurun_out/${TAG}_bench.log | cut -c1-300
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ism_ -s 3 -c 1 -o gpurun_out/${TAG}_prof_ism python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-sweep --e2e-steps 1 > gpurun_out/${TAG}_ncu.log 2>&1
tail -1 gpurun_out/${TAG}_ncu.log
