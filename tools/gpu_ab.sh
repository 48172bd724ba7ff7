cd $GRAFT_REPO_ROOT
python bench.py --steps 20000 --warmup 2000 --no-cpu --e2e-steps 0 > gpurun_out/ab_tma.json 2>&1
DK_NO_TMA=1 python bench.py --steps 20000 --warmup 2000 --no-cpu --e2e-steps 0 > gpurun_out/ab_notma.json 2>&1
CMD="python tools/profile_rollout.py --steps 1000 --launches 3"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:rollout_kernel -s 1 -c 1 -o gpurun_out/prof_rollout $CMD > gpurun_out/ncu.log 2>&1
DK_NO_TMA=1 ncu --set full --clock-control none --import-source on -k regex:rollout_kernel -s 1 -c 1 -o gpurun_out/prof_rollout_notma $CMD > gpurun_out/ncu2.log 2>&1
