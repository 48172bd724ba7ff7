cd $GRAFT_REPO_ROOT
timeout 900 python tools/parity_report.py > gpurun_out/parity.log 2>&1; echo "parity rc=$?" >> gpurun_out/parity.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
