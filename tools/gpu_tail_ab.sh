# Go1 tail / DR kernels after a change: their parity tests, tail timing, full bench line.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_locomotion.py tests/test_gpu_envstep.py -q -x > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ab_tests.log
timeout 300 python tools/exp_tail.py > gpurun_out/ab_tail.log 2>&1
timeout 900 python bench.py > gpurun_out/ab_bench.json 2> gpurun_out/ab_bench.err
echo done
