#!/bin/bash
cd ${GRAFT_REPO_ROOT:-$(dirname $0)/..}
O=gpurun_out/${TAG:-mlp}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_mlp.py tests/test_gpu_rollout.py -m gpu -q -s -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python tools/mlp_speed.py > $O/speed.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-tail --e2e-steps 1 > $O/bench.out 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mlp_tc_kernel -s 2 -c 1 -o $O/mlp python tools/mlp_speed.py > $O/ncu.log 2>&1; echo "ncu rc=$?" >> $O/pytest.log
