"""Go1 e2e (host buffers) vs chunk size and step count: python tools/go1_e2e_sweep.py"""
import sys, json, torch
sys.argv = ["bench.py"]
sys.path.insert(0, "."); import bench
from paper_2502_08844_b200 import go1env as G
args = bench.parse()
dev = torch.device("cuda", 0)
env = G.DeviceGo1Env(8192, G.Go1Config(), dtype="float32", device=0)
env.reset(seed=0)
res = []
for K in (200, 1000):
    for U in (5, 10, 20, 50):
        args.e2e_steps, args.unroll = K, U
        r = bench.measure_go1_e2e(env, args, dev, None, 1)
        res.append((K, U, r["value"]))
        print(K, U, "%.3e" % r["value"], flush=True)
