#!/bin/bash
# Round 2: physics parity + speed, f32 envstep/locomotion parity tests, rollout tests
cd ${GRAFT_REPO_ROOT:-$(dirname $0)/..}
mkdir -p gpurun_out/phys
timeout 900 python tools/phys_parity.py --n 8192 > gpurun_out/phys/parity.log 2>&1
timeout 300 python tools/phys_speed.py > gpurun_out/phys/speed.log 2>&1
timeout 300 python tools/phys_speed.py --full --worlds 8192 >> gpurun_out/phys/speed.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_envstep.py tests/test_gpu_locomotion.py tests/test_gpu_rollout.py -m gpu -q > gpurun_out/phys/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/phys/pytest.log
