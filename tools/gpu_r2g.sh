#!/bin/bash
# round-2: warp-parallel item setup — poly parity subset, setup sub-steps, small-call graph replay A/B, bench A/B
cd $GRAFT_REPO_ROOT
python -m pytest tests -q -m gpu -k "poly or cluster or graph or small or degenerate or batch" 2>&1 | tail -3 > gpurun_out/r2g_pytest.log
for c in cfg1 cfg2_2.0; do
GPURIR_LIB=build/phase.so python tools/phase_probe.py $c 0 > gpurun_out/r2g_phase_${c}.log 2>&1
echo "== $c"; python tools/phase_probe.py --parse gpurun_out/r2g_phase_${c}.log | grep -v "^  tile"
done > gpurun_out/r2g_phase.txt 2>&1
for r in 1 2; do for L in build/base.so paper_1810_11359_b200/libgpurir.so; do
  echo "== $L"; GPURIR_LIB=$L python tools/small_calls.py --reps 20 2>&1 | grep "split=  0" | grep "poly"
done; done > gpurun_out/r2g_small.txt 2>&1
bash tools/ab_bench.sh 3 build/base.so paper_1810_11359_b200/libgpurir.so > gpurun_out/r2g_ab.txt 2>&1
