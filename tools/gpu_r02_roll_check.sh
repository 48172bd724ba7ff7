cd $GRAFT_REPO_ROOT
O=gpurun_out/roll3; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_envstep.py tests/test_gpu_rollout.py tests/test_gpu_integration.py tests/test_gpu_dist_shards.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for t in cartpole-balance pendulum-swingup acrobot-swingup reacher-easy; do timeout 120 python tools/exp_rollout.py --task $t --worlds 1024,4096,8192 --tag solo_auto >> $O/speed.txt 2>&1; done
