# tensor-core MLP: tests, per-call device time (CUDA graph), optional ncu capture;
# VARIANTS="a b": build/variants/<v>.so timed beside the product build
cd ${GRAFT_REPO_ROOT:-$(dirname $0)/..}
O=gpurun_out/${TAG:-mlp2}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_mlp.py tests/test_gpu_rollout.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for v in product $VARIANTS; do
  if [ $v = product ]; then L=""; else L=build/variants/$v.so; fi
  echo "== $v" >> $O/speed.txt
  for k in value policy; do for r in 8192 16384; do DK_LIB_PATH=$L MLP_KIND=$k MLP_ROWS=$r timeout 120 python tools/prof_mlp_value.py >> $O/speed.txt 2>&1; done; done
done
if [ "${NCU:-1}" = 1 ]; then
MLP_KIND=${NCU_KIND:-value} timeout 600 ncu --set full --clock-control none --import-source on -k regex:mlp_tc_kernel -s 3 -c 1 -o $O/mlp_value python tools/prof_mlp_value.py > $O/ncu.log 2>&1
fi
