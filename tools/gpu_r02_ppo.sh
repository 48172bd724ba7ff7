#!/bin/bash
cd ${GRAFT_REPO_ROOT:-$(dirname $0)/..}
O=gpurun_out/${TAG:-ppo}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_mlp.py tests/test_gpu_rollout.py tests/test_gpu_ppo.py -m gpu -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-tail --e2e-steps 1 > $O/bench.out 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_ppo.csv python tools/prof_ppo.py > $O/ncu.log 2>&1; echo "ncu rc=$?" >> $O/pytest.log
