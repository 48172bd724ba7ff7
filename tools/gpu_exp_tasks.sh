# time variants (build/variants/*.so) on several tasks: bash tools/gpu_exp_tasks.sh v1 v2 ...
cd $GRAFT_REPO_ROOT
for t in ${TASKS:-cartpole-balance pendulum-swingup}; do
  for v in "$@"; do
    echo -n "$t " >> gpurun_out/exp.txt
    DK_LIB_PATH=build/variants/$v.so python tools/exp_rollout.py --task $t --worlds 8192 --steps ${K:-16000} --launches 3 >> gpurun_out/exp.txt 2>&1
  done
done
