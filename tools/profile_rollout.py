"""Small driver for ncu: a few rollout launches of the bench workload.

    python tools/profile_rollout.py [--task cartpole-balance] [--dtype float32]
        [--num-envs 8192] [--steps 1000] [--launches 3]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--task", default="cartpole-balance")
    ap.add_argument("--dtype", default="float32")
    ap.add_argument("--num-envs", type=int, default=8192)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--launches", type=int, default=3)
    a = ap.parse_args()
    import torch

    import paper_2502_08844_b200 as dk

    env = dk.DeviceBatchEnv(dk.EnvConfig(task=a.task), a.num_envs, dtype=a.dtype)
    env.reset(seed=0)
    acts = torch.rand((a.steps, a.num_envs, env.action_dim), device="cuda",
                      dtype=env.dtype) * 2 - 1
    out = env._outputs((a.steps,), True)
    for _ in range(a.launches):
        env.rollout(acts, with_info=True, out=out)
    env.check()
    torch.cuda.synchronize()
    print("ok", env.kernel_launches)


if __name__ == "__main__":
    main()
