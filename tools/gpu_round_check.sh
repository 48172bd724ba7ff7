# Full GPU check: test suite, smoke, default bench line, pixel_normalize ncu capture.
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 300 python tools/exp_pixnorm.py 8192 > gpurun_out/pixnorm_plain.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:pixnorm -c 2 -o gpurun_out/pixnorm_cur -f python tools/exp_pixnorm.py 8192 > gpurun_out/pixnorm_ncu.log 2>&1
echo done
