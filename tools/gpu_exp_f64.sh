# f64 rollout A/B: speed per task (product vs variants) + the f64 parity tests
cd ${GRAFT_REPO_ROOT:-$(dirname $0)/..}
O=gpurun_out/${TAG:-f64ab}; mkdir -p $O
for v in product "$@"; do
  if [ $v = product ]; then L=""; else L=build/variants/$v.so; fi
  for t in cartpole-balance pendulum-swingup acrobot-swingup reacher-easy; do
    DK_LIB_PATH=$L timeout 120 python tools/exp_rollout.py --task $t --dtype float64 --worlds 1024,8192 --tag $v >> $O/speed.txt 2>&1
  done
done
timeout 900 python -m pytest tests/test_gpu_envstep.py tests/test_gpu_rollout.py tests/test_gpu_integration.py tests/test_gpu_locomotion.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
