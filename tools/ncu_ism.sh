cd /root/repo
python -c "import __graft_entry__ as g; g.build()"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ism_ -s 3 -c 1 -o gpurun_out/${1:-x}_prof_ism python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/${1:-x}_ncu.log 2>&1
tail -2 gpurun_out/${1:-x}_ncu.log
