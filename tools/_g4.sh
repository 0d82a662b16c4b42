cd $GRAFT_REPO_ROOT
python tools/diag_rigid.py > gpurun_out/g4_diag_new.txt 2>&1
GPURIR_LIB=build/old_r1.so python tools/diag_rigid.py > gpurun_out/g4_diag_old.txt 2>&1
python tools/small_calls.py > gpurun_out/g4_small.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g4_small_ncu.csv python tools/small_calls.py --reps 3 > /dev/null 2>&1
tail -3 gpurun_out/g4_small_ncu.csv
