cd $GRAFT_REPO_ROOT
python bench.py --steps 20000 --warmup 2000 --no-cpu --e2e-steps 0 --no-tail --no-extra > gpurun_out/exp32.json 2>&1
