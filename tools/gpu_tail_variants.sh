# Time the Go1 tail under library variants built by tools/exp_variants.sh
# (tools/gpu_tail_variants.sh v1 v2 ...), after the tail's parity tests.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_locomotion.py -q -x > gpurun_out/tailvar_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/tailvar_tests.log
for v in "$@"; do
  echo "== $v" >> gpurun_out/tailvar.log
  DK_LIB_PATH=build/variants/$v.so timeout 300 python tools/exp_tail.py >> gpurun_out/tailvar.log 2>&1
done
echo done
