# Build experimental variants of the library here (cross-compile), e.g.
#   bash tools/exp_variants.sh build base "" rolemap "-DDK_EXP_ROLEMAP"
# and time them on the GPU box:
#   bash tools/exp_variants.sh run base rolemap        (inside gpurun)
set -e
cd ${GRAFT_REPO_ROOT:-$(dirname $0)/..}
mode=$1; shift
if [ "$mode" = build ]; then
  while [ $# -gt 0 ]; do
    name=$1; flags=$2; shift 2
    DK_NVCC_EXTRA="$flags" DK_LIB_OUT=build/variants/$name.so DK_OBJ_DIR=build/variants/obj_$name \
      python -m paper_2502_08844_b200.build --force
  done
else
  for name in "$@"; do
    for dt in float32; do
      DK_LIB_PATH=build/variants/$name.so python tools/exp_rollout.py --dtype $dt ${EXP_ARGS} >> gpurun_out/exp.txt 2>&1 || echo "$name failed" >> gpurun_out/exp.txt
    done
  done
fi
