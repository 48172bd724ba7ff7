# pixel_normalize after a change: pixel parity tests, then timing of the product
# library against variants built by tools/exp_variants.sh (args).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pixels.py -q -x > gpurun_out/pn_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/pn_tests.log
for round in 1 2; do
  echo "== product" >> gpurun_out/pn_ab.log
  timeout 300 python tools/exp_pixnorm.py 8192 >> gpurun_out/pn_ab.log 2>&1
  timeout 300 python tools/exp_pixnorm.py 8192 env >> gpurun_out/pn_ab.log 2>&1
  for v in "$@"; do
    echo "== $v" >> gpurun_out/pn_ab.log
    DK_LIB_PATH=build/variants/$v.so timeout 300 python tools/exp_pixnorm.py 8192 >> gpurun_out/pn_ab.log 2>&1
    DK_LIB_PATH=build/variants/$v.so timeout 300 python tools/exp_pixnorm.py 8192 env >> gpurun_out/pn_ab.log 2>&1
  done
done
echo done
