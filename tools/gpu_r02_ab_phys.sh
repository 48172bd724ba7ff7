#!/bin/bash
# A/B of physics-kernel variants: DK_LIB_PATH=build/variants/<name>.so; the
# physics / Go1 GPU tests run on each variant too (TEST_VARIANTS=1)
cd ${GRAFT_REPO_ROOT:-$(dirname $0)/..}
O=gpurun_out/${PERF_TAG:-abphys}; mkdir -p $O
for v in product "$@"; do
  if [ $v = product ]; then L=""; else L=build/variants/$v.so; fi
  echo "== $v" >> $O/speed.log
  DK_LIB_PATH=$L timeout 300 python tools/phys_speed.py --worlds 8192,65536 --dtypes float32,float64 >> $O/speed.log 2>&1
  DK_LIB_PATH=$L timeout 300 python tools/go1_speed.py --worlds 8192 >> $O/speed.log 2>&1
  if [ "${TEST_VARIANTS:-0}" = 1 ] || [ $v = product ]; then
    DK_LIB_PATH=$L timeout 900 python -m pytest tests/test_gpu_go1env.py tests/test_gpu_physics.py -m gpu -q -x > $O/pytest_$v.log 2>&1; echo "pytest rc=$?" >> $O/pytest_$v.log
  fi
done
