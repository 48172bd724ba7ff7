cd $GRAFT_REPO_ROOT
python bench.py --steps 20000 --warmup 2000 --no-cpu --e2e-steps 0 > gpurun_out/b32.json 2>&1
python bench.py --steps 20000 --warmup 2000 --no-cpu --e2e-steps 0 --dtype float64 > gpurun_out/b64.json 2>&1
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
