# Time the Go1 tail under library variants (build/variants/<v>.so) against the
# product build, after the tail's parity tests on each
cd ${GRAFT_REPO_ROOT:-$(dirname $0)/..}
O=gpurun_out/${TAG:-tailvar}; mkdir -p $O
for v in product "$@"; do
  if [ $v = product ]; then L=""; else L=build/variants/$v.so; fi
  DK_LIB_PATH=$L timeout 900 python -m pytest tests/test_gpu_locomotion.py -q -x > $O/tests_$v.log 2>&1; echo "tests rc=$?" >> $O/tests_$v.log
  echo "== $v" >> $O/tail.log
  DK_LIB_PATH=$L timeout 300 python tools/exp_tail.py >> $O/tail.log 2>&1
done
