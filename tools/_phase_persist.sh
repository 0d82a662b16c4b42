cd $GRAFT_REPO_ROOT
GPURIR_LIB=build/phase.so timeout 300 python bench.py --no-cpu-baseline --no-sweep --ab-lib --e2e-steps 1 --steps 3 --warmup 3 2>&1 | grep "^PTL" | tail -8
