# physics parity report (+ Go1 / physics GPU tests, Go1 speed) for the product
# build or a variant (VARIANT=<name>: build/variants/<name>.so)
cd ${GRAFT_REPO_ROOT:-$(dirname $0)/..}
O=gpurun_out/${TAG:-pp}; mkdir -p $O
if [ -n "$VARIANT" ]; then export DK_LIB_PATH=build/variants/$VARIANT.so; fi
timeout 900 python tools/phys_parity.py --out $O/phys_parity.json > $O/pp.log 2>&1; echo "rc=$?" >> $O/pp.log
timeout 900 python -m pytest tests/test_gpu_go1env.py tests/test_gpu_physics.py -m gpu -q -s > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 300 python tools/go1_speed.py --worlds 1024,8192,65536 > $O/speed.log 2>&1
