cd $GRAFT_REPO_ROOT
for tl in 1 2; do
  DK_TILES=$tl python bench.py --steps 20000 --warmup 2000 --no-cpu --e2e-steps 0 --no-tail > gpurun_out/ab_tl$tl.json 2>&1
  DK_TILES=$tl python bench.py --steps 20000 --warmup 2000 --no-cpu --e2e-steps 0 --no-tail --dtype float64 > gpurun_out/ab64_tl$tl.json 2>&1
done
DK_TILES=2 timeout 900 python -m pytest tests/test_gpu_envstep.py -m gpu -q -x > gpurun_out/pytest_gpu_tl2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_tl2.log
