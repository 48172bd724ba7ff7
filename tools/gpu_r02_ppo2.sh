# PPO rollout: GPU tests, live kernel profile, bench leg
cd ${GRAFT_REPO_ROOT:-$(dirname $0)/..}
O=gpurun_out/${TAG:-ppo2}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_rollout.py tests/test_gpu_ppo.py tests/test_gpu_mlp.py tests/test_gpu_dist_normalizer.py tests/test_gpu_integration.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 600 python tools/prof_ppo_live.py > $O/prof.txt 2>&1
timeout 600 python -c "
import bench, argparse, torch, json
a = argparse.Namespace(num_envs=8192, analytic_task='cartpole-balance')
print(json.dumps(bench.bench_ppo_rollout(a, torch.device('cuda', 0))))
" > $O/ppo_bench.json 2> $O/ppo_bench.err
