#!/bin/bash
cd $GRAFT_REPO_ROOT
GPURIR_POLY_CL_S=1 python -m pytest tests -q -m gpu -k "poly or cluster or graph or small or degenerate or cfg2 or cfg1" 2>&1 | tail -4 > gpurun_out/r2k_pytest.log
for r in 1 2; do
  echo "== default"; python tools/small_calls.py --reps 20 2>&1 | grep "split=  0" | grep "poly"
  echo "== S=1 1024"; GPURIR_POLY_CL_S=1 python tools/small_calls.py --reps 20 2>&1 | grep "split=  0" | grep "poly"
  echo "== S=1 512"; GPURIR_POLY_CL_S=1 GPURIR_POLY_CL_THREADS=512 python tools/small_calls.py --reps 20 2>&1 | grep "split=  0" | grep "poly"
done > gpurun_out/r2k_small.txt 2>&1
for c in cfg1 cfg2_2.0; do
GPURIR_POLY_CL_S=1 GPURIR_LIB=build/phase.so python tools/phase_probe.py $c 0 > gpurun_out/r2k_phase_$c.log 2>&1
echo "== $c S=1"; python tools/phase_probe.py --parse gpurun_out/r2k_phase_$c.log
done > gpurun_out/r2k_phase.txt 2>&1
