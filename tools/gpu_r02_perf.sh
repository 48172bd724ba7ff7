#!/bin/bash
# physics / go1 kernel perf iteration: tests, speed, one ncu capture
cd ${GRAFT_REPO_ROOT:-$(dirname $0)/..}
O=gpurun_out/${PERF_TAG:-perf}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_go1env.py tests/test_gpu_physics.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 300 python tools/phys_speed.py --worlds 1024,8192,65536 > $O/speed.log 2>&1
timeout 300 python tools/go1_speed.py --worlds 1024,4096,8192,65536 >> $O/speed.log 2>&1
PROF_K=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:go1_env_kernel -s 1 -c 1 -o $O/go1_env python tools/prof_go1.py > $O/ncu_go1.log 2>&1; echo "ncu go1 rc=$?" >> $O/rc.txt
