# analytic rollout kernel: the env / rollout / integration GPU tests, then the
# speed of every task at 1K-64K worlds for the product and VARIANTS
cd ${GRAFT_REPO_ROOT:-$(dirname $0)/..}
O=gpurun_out/${TAG:-roll2}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_envstep.py tests/test_gpu_rollout.py tests/test_gpu_integration.py tests/test_gpu_dist_shards.py tests/test_gpu_pixels.py tests/test_gpu_serve.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for v in product $VARIANTS; do
  if [ $v = product ]; then L=""; else L=build/variants/$v.so; fi
  for dt in float32 float64; do for t in cartpole-balance pendulum-swingup acrobot-swingup reacher-easy; do
    DK_LIB_PATH=$L timeout 120 python tools/exp_rollout.py --task $t --dtype $dt --worlds 1024,4096,8192,65536 --tag $v >> $O/speed.txt 2>&1
  done; done
done
