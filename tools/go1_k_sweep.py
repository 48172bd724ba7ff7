"""Go1 env kernel time per control step vs steps fused per launch (K; the PPO
rollout steps with K = 1).  python tools/go1_k_sweep.py
r02: 116.6 / 112.3 / 109.4 / 106.5 / 104.3 us per step at K = 1 / 2 / 4 / 10 / 20
(8192 worlds, fresh from reset)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2502_08844_b200 import go1env as G

    n = 8192
    env = G.DeviceGo1Env(n, G.Go1Config(), dtype="float32")
    env.reset(seed=0)
    res = {}
    for K in (1, 2, 4, 10, 20):
        act = torch.rand(K, n, 12, device="cuda") * 2 - 1
        for _ in range(3):
            env.rollout(act)
        torch.cuda.synchronize()
        reps = max(2, 40 // K)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            env.rollout(act)
        b.record()
        torch.cuda.synchronize()
        res[f"K{K}_us_per_step"] = a.elapsed_time(b) * 1e3 / (reps * K)
    env.check()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
