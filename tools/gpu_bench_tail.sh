cd $GRAFT_REPO_ROOT
python bench.py --steps 20000 --warmup 2000 --cpu-seconds 4 > gpurun_out/bench.json 2> gpurun_out/bench.err
CMD="python tools/profile_tail.py"
$CMD > gpurun_out/prof_tail_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:loco_tail_kernel -s 1 -c 1 -o gpurun_out/prof_tail $CMD > gpurun_out/ncu_tail.log 2>&1
echo done
