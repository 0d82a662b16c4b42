#!/bin/bash
# build libgpurir.so (+ the phase-timing variant) and fail loudly if either did not rebuild
cd "$(dirname "$0")/.."
python -c "from paper_1810_11359_b200 import build as B; B.build()" > /tmp/build.log 2>&1 || { grep -i error /tmp/build.log | head; exit 1; }
[ "${1}" == "phase" ] && { bash tools/build_variant.sh phase -DGPURIR_PHASE_TIMING > /tmp/build_v.log 2>&1 || { grep -i error /tmp/build_v.log | head; exit 1; }; }
ls -la --time-style=+%T paper_1810_11359_b200/libgpurir.so | awk '{print "built", $6, $7}'
