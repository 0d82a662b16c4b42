#!/bin/bash
cd $GRAFT_REPO_ROOT
GPURIR_PLAN_TIMING=1 python tools/prof_cfg5_host.py > gpurun_out/r2n_cfg5_host.txt 2>&1
GPURIR_BENCH_DEBUG=1 python bench.py --workload cfg5 --no-cpu-baseline > gpurun_out/r2n_cfg5.log 2>&1
GPURIR_BENCH_DEBUG=1 python bench.py --workload cfg5 --no-cpu-baseline > gpurun_out/r2n_cfg5b.log 2>&1
