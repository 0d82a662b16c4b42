cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/g5_pytest_gpu.log 2>&1; tail -3 gpurun_out/g5_pytest_gpu.log
bash tools/sanitize.sh
