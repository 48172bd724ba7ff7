cd $GRAFT_REPO_ROOT
python bench.py --steps 20000 --warmup 2000 --no-cpu --e2e-steps 0 --no-tail --no-extra > gpurun_out/q32.json 2>&1
python bench.py --steps 20000 --warmup 2000 --no-cpu --e2e-steps 0 --no-tail --no-extra --dtype float64 > gpurun_out/q64.json 2>&1
timeout 900 python -m pytest tests/test_gpu_envstep.py -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
