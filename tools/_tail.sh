cd $GRAFT_REPO_ROOT
echo "== fused tail (default)"; python tools/small_calls.py --reps 20 | grep -E "cfg2_2.0|cfg4|cfg2_0.7" | grep "split=  0"
echo "== tail_kernel (GPURIR_FUSE_TAIL=0)"; GPURIR_FUSE_TAIL=0 python tools/small_calls.py --reps 20 | grep -E "cfg2_2.0|cfg4|cfg2_0.7" | grep "split=  0"
ncu --set full --clock-control none --import-source on -k regex:tail_kernel -s 3 -c 1 -o gpurun_out/tail_v2 python bench.py --mode fp32 --steps 1 --warmup 3 --no-cpu-baseline --no-sweep --e2e-steps 1 > /dev/null 2>&1
ls gpurun_out/tail_v2*
