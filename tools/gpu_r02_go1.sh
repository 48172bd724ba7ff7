#!/bin/bash
cd ${GRAFT_REPO_ROOT:-$(dirname $0)/..}
mkdir -p gpurun_out/go1
timeout 900 python -m pytest tests/test_gpu_go1env.py tests/test_gpu_physics.py tests/test_gpu_rollout.py -m gpu -q -x > gpurun_out/go1/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/go1/pytest.log
timeout 300 python tools/go1_speed.py > gpurun_out/go1/speed.log 2>&1
