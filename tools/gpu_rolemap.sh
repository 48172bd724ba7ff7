# analytic rollout warp-role placement A/B: product vs build/variants/$V.so, f32 / f64, all tasks
cd ${GRAFT_REPO_ROOT:-$(dirname $0)/..}
O=gpurun_out/${TAG:-rolemap}; mkdir -p $O
for t in cartpole-balance pendulum-swingup acrobot-swingup reacher-easy; do
 for dt in float32 float64; do
  for v in product ${V:-rolemap2} product ${V:-rolemap2}; do
   if [ $v = product ]; then L=""; else L=build/variants/$v.so; fi
   echo "== $v $t $dt" >> $O/out.txt
   DK_LIB_PATH=$L timeout 120 python tools/exp_rollout.py --task $t --dtype $dt --worlds 1024,8192 >> $O/out.txt 2>&1
  done
 done
done
