#!/bin/bash
cd ${GRAFT_REPO_ROOT:-$(dirname $0)/..}
mkdir -p gpurun_out/phys2
timeout 1200 python tools/phys_parity.py --n 8192 --out gpurun_out/phys2/parity.json > gpurun_out/phys2/parity.log 2>&1
timeout 300 python tools/phys_speed.py --full --worlds 8192 > gpurun_out/phys2/speed.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_envstep.py tests/test_gpu_locomotion.py -m gpu -q > gpurun_out/phys2/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/phys2/pytest.log
