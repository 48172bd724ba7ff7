# Round-end refresh: GPU tests, smoke, default bench line, reference arm, launch lists.
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_tests.log 2>&1; echo "rc=$?" >> gpurun_out/final_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/final_smoke.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/final_clocks.csv &
SMI=$!
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
kill $SMI
timeout 600 python bench.py --impl reference > gpurun_out/final_reference.json 2> gpurun_out/final_reference.err
BENCH="python bench.py --steps 20000 --warmup 2000 --no-cpu --e2e-steps 0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv $BENCH > gpurun_out/final_ncu.log 2>&1
HEAD="python bench.py --steps 20000 --warmup 2000 --no-cpu --e2e-steps 0 --no-tail --no-extra"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches_headline.csv $HEAD > gpurun_out/final_ncu_head.log 2>&1
echo done
