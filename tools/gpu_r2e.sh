#!/bin/bash
# round-2 final evidence: smoke, all GPU tests, default bench (sweep), trajectory and cfg5 benches, launch lists,
# ncu --set full of the polyphase kernel (bench step) and of the tensor-core trajectory kernel
TAG=${1:-r2e}
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -2 gpurun_out/${TAG}_smoke.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/${TAG}_pytest_gpu.log 2>&1; tail -1 gpurun_out/${TAG}_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; tail -1 gpurun_out/${TAG}_bench.log | cut -c1-200
timeout 600 python bench.py --workload trajectory > gpurun_out/${TAG}_bench_traj.log 2>&1; tail -1 gpurun_out/${TAG}_bench_traj.log | cut -c1-200
timeout 600 python bench.py --workload cfg5 > gpurun_out/${TAG}_bench_cfg5.log 2>&1; tail -1 gpurun_out/${TAG}_bench_cfg5.log | cut -c1-200
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${TAG}_bench_ref.log 2>&1; tail -1 gpurun_out/${TAG}_bench_ref.log | cut -c1-200
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sweep --e2e-steps 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_traj_launches.csv python bench.py --workload trajectory --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ism_poly -s 3 -c 1 -o gpurun_out/${TAG}_poly python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-sweep --e2e-steps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:traj_tc -s 2 -c 1 -o gpurun_out/${TAG}_traj_tc python tools/prof_traj.py 0 > /dev/null 2>&1
ls gpurun_out/ | grep ${TAG}
