cd $GRAFT_REPO_ROOT
for c in cfg1 cfg2_2.0; do
GPURIR_LIB=build/phase.so python tools/phase_probe.py $c 0 > gpurun_out/phase_${c}_0.log 2>&1
echo "== $c"; python tools/phase_probe.py --parse gpurun_out/phase_${c}_0.log | grep -v "^  tile"
done
python tools/small_calls.py --reps 20
echo "--- 512-thread cluster CTAs"
GPURIR_POLY_CL_THREADS=512 python tools/small_calls.py --reps 20 | grep "split=  0"
