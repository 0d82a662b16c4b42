#!/bin/bash
# A/B the ISM bench across variant libraries (run under gpurun): tools/ab_bench.sh <reps> lib1.so lib2.so ...
cd "$(dirname "$0")/.."
REPS=$1; shift
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in $(seq 1 $REPS); do
  for L in "$@"; do
    v=$(GPURIR_LIB=$L timeout 300 python bench.py --no-cpu-baseline --no-sweep --ab-lib --e2e-steps 2 --steps 10 2>/dev/null | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print(f\"{d['value']:.0f} ms_per_step={d['ms_per_step']:.4f} parity={d.get('parity',{}).get('max_err_over_peak')}\")")
    echo "$L $v"
  done
done
