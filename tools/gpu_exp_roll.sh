# rollout-kernel experiments: A/B of variants and an ncu capture at 1024 worlds
cd ${GRAFT_REPO_ROOT:-$(dirname $0)/..}
O=gpurun_out/${TAG:-roll}; mkdir -p $O
for v in product "$@"; do
  if [ $v = product ]; then L=""; else L=build/variants/$v.so; fi
  for t in cartpole-balance pendulum-swingup; do
    DK_LIB_PATH=$L timeout 120 python tools/exp_rollout.py --task $t --worlds 1024,4096,8192,65536 --tag $v >> $O/speed.txt 2>&1
  done
done
if [ "${NCU:-0}" = 1 ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rollout_kernel -s 3 -c 1 -o $O/roll1024 python tools/exp_rollout.py --task cartpole-balance --worlds 1024 --launches 4 > $O/ncu1024.log 2>&1
fi
