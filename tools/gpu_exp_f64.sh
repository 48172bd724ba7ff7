cd $GRAFT_REPO_ROOT
for v in "$@"; do
  echo -n "f64 " >> gpurun_out/exp.txt
  DK_LIB_PATH=build/variants/$v.so python tools/exp_rollout.py --dtype float64 --worlds 8192 --steps 4000 --launches 3 >> gpurun_out/exp.txt 2>&1
done
