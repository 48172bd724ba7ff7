# tensor-core MLP A/B variants (build/variants/<v>.so from tools/exp_variants.sh build),
# per-call device time from CUDA-graph replays: VARIANTS="a b" bash tools/gpu_mlp_variants.sh
cd ${GRAFT_REPO_ROOT:-$(dirname $0)/..}
O=gpurun_out/${TAG:-mlpvar}; mkdir -p $O
for v in product $VARIANTS; do
  if [ $v = product ]; then L=""; else L=build/variants/$v.so; fi
  echo "== $v" >> $O/speed.txt
  for r in 8192 245760; do DK_LIB_PATH=$L MLP_KIND=value MLP_ROWS=$r timeout 120 python tools/prof_mlp_value.py >> $O/speed.txt 2>&1; done
  DK_LIB_PATH=$L MLP_KIND=value MLP_DIN=75 MLP_ROWS=245760 timeout 120 python tools/prof_mlp_value.py >> $O/speed.txt 2>&1
  DK_LIB_PATH=$L MLP_KIND=policy MLP_ROWS=8192 timeout 120 python tools/prof_mlp_value.py >> $O/speed.txt 2>&1
  DK_LIB_PATH=$L MLP_KIND=policy MLP_DIN=56 MLP_ROWS=8192 timeout 120 python tools/prof_mlp_value.py >> $O/speed.txt 2>&1
done
