#!/bin/bash
# Round 2 full check: the driver's bench command + reference arm, the whole GPU
# test suite, smoke, ncu launch list of the bench and full captures of the Go1 kernels
cd ${GRAFT_REPO_ROOT:-$(dirname $0)/..}
O=gpurun_out/${TAG:-full}; mkdir -p $O
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > $O/clocks.csv &
CLK=$!
timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench.out 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
kill $CLK
timeout 900 python3 bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/ref.out 2> $O/ref.err; echo "ref rc=$?" >> $O/rc.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
if [ "${NCU:-1}" = 1 ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv python3 bench.py --gpus 1 --steps 20 --warmup 5 --no-extra --no-cpu --no-tail > $O/ncu_launches.log 2>&1; echo "ncu launches rc=$?" >> $O/rc.txt
PROF_K=20 timeout 900 ncu --set full --clock-control none --import-source on -k regex:go1_env_kernel -s 1 -c 1 -o $O/go1_env python tools/prof_go1.py > $O/ncu_go1.log 2>&1; echo "ncu go1 rc=$?" >> $O/rc.txt
PROF_K=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:phys_kernel -s 1 -c 1 -o $O/phys python tools/prof_go1.py > $O/ncu_phys.log 2>&1; echo "ncu phys rc=$?" >> $O/rc.txt
fi
if [ "${NCU:-1}" = 1 ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mlp_tc_kernel -s 2 -c 1 -o $O/mlp python tools/mlp_speed.py > $O/ncu_mlp.log 2>&1; echo "ncu mlp rc=$?" >> $O/rc.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_ppo.csv python tools/prof_ppo.py > $O/ncu_ppo.log 2>&1; echo "ncu ppo rc=$?" >> $O/rc.txt
fi
