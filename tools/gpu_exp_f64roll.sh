# ncu capture of the f64 cartpole rollout kernel at 8192 worlds (source-level)
cd ${GRAFT_REPO_ROOT:-$(dirname $0)/..}
O=gpurun_out/${TAG:-f64roll}; mkdir -p $O
timeout 120 python tools/exp_rollout.py --task cartpole-balance --dtype float64 --worlds 1024,8192 > $O/speed.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rollout_kernel -s 3 -c 1 -o $O/roll64 python tools/exp_rollout.py --task cartpole-balance --dtype float64 --worlds 8192 --launches 4 > $O/ncu.log 2>&1
