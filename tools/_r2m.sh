#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m pytest tests -q -m gpu -k "batch or shard or cfg5 or workspace or room" 2>&1 | tail -3 > gpurun_out/r2m_pytest.log
python tools/prof_cfg5_host.py > gpurun_out/r2m_cfg5_host.txt 2>&1
GPURIR_PLAN_THREADS=1 python tools/prof_cfg5_host.py 2>&1 | head -3 | sed 's/^/serial: /' >> gpurun_out/r2m_cfg5_host.txt
GPURIR_BENCH_DEBUG=1 python bench.py --workload cfg5 --no-cpu-baseline > gpurun_out/r2m_cfg5.log 2>&1
