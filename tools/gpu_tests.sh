cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -k "${1:-.}" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
