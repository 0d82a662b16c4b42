cd $GRAFT_REPO_ROOT
for S in 4 8 16; do for T in 1024 512; do echo "== S=$S threads=$T"; GPURIR_POLY_CL_S=$S GPURIR_POLY_CL_THREADS=$T python tools/small_calls.py --reps 20 | grep "split=  0" | grep poly | cut -c1-20,95-130; done; done
