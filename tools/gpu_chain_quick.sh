# chain microbenchmark + quick bench (f32/f64) + envstep GPU parity tests
cd $GRAFT_REPO_ROOT
./tools/micro/chainbench > gpurun_out/chainbench.txt 2>&1
bash tools/gpu_quick.sh
