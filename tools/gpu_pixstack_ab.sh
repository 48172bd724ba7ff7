# A/B of the pixel stack kernel's CTA shape (variants built by tools/exp_variants.sh)
cd ${GRAFT_REPO_ROOT:-$(dirname $0)/..}
python -m pytest tests/test_gpu_pixels.py tests/test_gpu_rollout.py tests/test_gpu_serve.py -q -x > gpurun_out/ab_tests.log 2>&1
echo "tests: $(tail -1 gpurun_out/ab_tests.log)"
echo "base: $(python tools/exp_pixstack.py)"
for v in "$@"; do
  echo "$v: $(DK_LIB_PATH=build/variants/$v.so python tools/exp_pixstack.py)"
  DK_LIB_PATH=build/variants/$v.so python -m pytest tests/test_gpu_pixels.py -q -x 2>&1 | tail -1
done
