# Round profile capture: bench line, ncu launch list of the same command,
# and one full ncu capture of the rollout kernel (bench workload shape).
cd $GRAFT_REPO_ROOT
BENCH="python bench.py --steps 20000 --warmup 2000 --no-cpu --e2e-steps 0"
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks.csv &
SMI=$!
$BENCH > gpurun_out/prof_bench.json 2> gpurun_out/prof_bench.err
kill $SMI
$BENCH > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $BENCH > gpurun_out/ncu_launches.log 2>&1
# the headline timed region alone (no extras): the rollout kernel's share of the step
HEAD="python bench.py --steps 20000 --warmup 2000 --no-cpu --e2e-steps 0 --no-tail --no-extra"
$HEAD > gpurun_out/plain_head.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_headline.csv $HEAD > gpurun_out/ncu_launches_head.log 2>&1
CMD="python tools/profile_rollout.py --steps 1000 --launches 3"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:rollout_kernel -s 1 -c 1 -o gpurun_out/prof_rollout $CMD > gpurun_out/ncu.log 2>&1
CMD64="python tools/profile_rollout.py --steps 1000 --launches 3 --dtype float64"
$CMD64 > gpurun_out/prof_plain64.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:rollout_kernel -s 1 -c 1 -o gpurun_out/prof_rollout64 $CMD64 > gpurun_out/ncu64.log 2>&1
echo done
