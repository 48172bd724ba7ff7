# time the in-tree library at several K (steps per launch)
cd $GRAFT_REPO_ROOT
for k in ${KS:-1000 16000}; do python tools/exp_rollout.py --worlds ${WORLDS:-8192} --steps $k --launches 10 >> gpurun_out/exp.txt 2>&1; done
