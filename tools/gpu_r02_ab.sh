#!/bin/bash
# Round 2: f32 accuracy A/B (parity at the 1e-3 floor + throughput per build)
# and the gated --steps 20 headline.   Run inside gpurun.
cd ${GRAFT_REPO_ROOT:-$(dirname $0)/..}
mkdir -p gpurun_out/ab
timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --no-extra --no-cpu --e2e-steps 0 > gpurun_out/ab/bench20.json 2> gpurun_out/ab/bench20.err
timeout 300 python bench.py --gpus 1 --steps 20000 --warmup 3000 --no-extra --no-cpu --e2e-steps 0 > gpurun_out/ab/bench20k.json 2>> gpurun_out/ab/bench20.err
for v in product faithful sincos div tol order; do
  if [ $v = product ]; then L=""; else L=build/variants/$v.so; fi
  DK_LIB_PATH=$L timeout 600 python tools/parity_report.py --dtypes float32 --tag $v --out gpurun_out/ab/parity_$v.json > gpurun_out/ab/parity_$v.log 2>&1
  for t in cartpole-balance pendulum-swingup acrobot-swingup reacher-easy; do
    DK_LIB_PATH=$L timeout 120 python tools/exp_rollout.py --task $t --worlds 1024,8192 --tag $v >> gpurun_out/ab/speed.txt 2>&1
  done
done
timeout 900 python -m pytest tests/test_gpu_rollout.py tests/test_gpu_integration.py -m gpu -q -x > gpurun_out/ab/pytest_rollout.log 2>&1; echo "rc=$?" >> gpurun_out/ab/pytest_rollout.log
