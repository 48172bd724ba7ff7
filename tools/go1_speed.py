"""Time the fused Go1 joystick env (DeviceGo1Env.rollout): control steps/s and
physics steps/s at several world counts.  Not a bench line.

    python tools/go1_speed.py [--worlds 1024,8192,65536] [--K 50]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--worlds", default="1024,8192,65536")
    ap.add_argument("--K", type=int, default=50)
    ap.add_argument("--dtypes", default="float32,float64")
    a = ap.parse_args()
    import torch

    from paper_2502_08844_b200 import go1env as G

    for dt in a.dtypes.split(","):
        res = []
        for n in [int(x) for x in a.worlds.split(",")]:
            env = G.DeviceGo1Env(n, G.Go1Config(), dtype=dt)
            env.reset(seed=0)
            acts = torch.rand((a.K, n, 12), device="cuda", dtype=env.dtype) * 2 - 1
            out = env.outputs(a.K)
            env.rollout(acts, out=out)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            reps = 3
            for _ in range(reps):
                env.rollout(acts, out=out)
            e1.record()
            torch.cuda.synchronize()
            env.check()
            ms = e0.elapsed_time(e1) / reps
            ctrl = n * a.K / (ms / 1e3)
            res.append(f"{n}:{ctrl:.3g}ctrl/s={ctrl * 5:.3g}phys/s({ms:.2f}ms/{a.K})")
            env.close()
        print("go1env", dt, " ".join(res), flush=True)


if __name__ == "__main__":
    main()
