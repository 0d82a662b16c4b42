#!/bin/bash
cd $GRAFT_REPO_ROOT
for r in 1 2 3; do GPURIR_BENCH_DEBUG=1 python bench.py --workload cfg5 --no-cpu-baseline > gpurun_out/r2o_cfg5_$r.log 2>&1; done
python -m pytest tests -q -m gpu -k "batch or shard or cfg5 or workspace or room" 2>&1 | tail -1 > gpurun_out/r2o_pytest.log
