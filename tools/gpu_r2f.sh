#!/bin/bash
# round-2 check: CUDA-graph tests in fresh processes (scratch rings grown together) + cfg1 setup sub-step probe
cd $GRAFT_REPO_ROOT
python -m pytest tests -q -m gpu -k "test_small_call_cuda_graph_replay" 2>&1 | tail -3 > gpurun_out/r2f_graph.log
python -m pytest tests -q -m gpu -k "graph or trajectory" 2>&1 | tail -3 >> gpurun_out/r2f_graph.log
for c in cfg1 cfg2_2.0; do
GPURIR_LIB=build/phase.so python tools/phase_probe.py $c 0 > gpurun_out/r2f_phase_${c}.log 2>&1
echo "== $c"; python tools/phase_probe.py --parse gpurun_out/r2f_phase_${c}.log | grep -v "^  tile"
done > gpurun_out/r2f_phase.txt 2>&1
