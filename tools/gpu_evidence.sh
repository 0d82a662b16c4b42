cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python tools/parity_report.py > gpurun_out/${TAG:-v27}_parity.txt 2>&1; tail -3 gpurun_out/${TAG:-v27}_parity.txt
timeout 1200 python tools/sweep.py > gpurun_out/${TAG:-v27}_sweep.jsonl 2> gpurun_out/${TAG:-v27}_sweep.err; wc -l gpurun_out/${TAG:-v27}_sweep.jsonl
timeout 600 python bench.py --workload trajectory --no-cpu-baseline > gpurun_out/${TAG:-v27}_traj.log 2>&1; tail -1 gpurun_out/${TAG:-v27}_traj.log | cut -c1-300
