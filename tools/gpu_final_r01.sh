# End-of-round check: GPU tests, smoke, default bench with clocks, reference arm,
# and the ncu launch list of the default bench command.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/fin_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/fin_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fin_smoke.log 2>&1
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/fin_clocks.csv &
SMI=$!
timeout 900 python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err
kill $SMI
timeout 600 python bench.py --impl reference > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches.csv \
  python bench.py --steps 20000 --warmup 2000 --no-cpu --e2e-steps 0 > gpurun_out/fin_ncu.log 2>&1
echo done
