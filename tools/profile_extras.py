"""ncu driver for the widened kernels: pixel stack, GAE, normaliser update.
python tools/profile_extras.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2502_08844_b200 as dk
    from paper_2502_08844_b200 import ppo as P

    n = 8192
    env = dk.DeviceBatchEnv(dk.EnvConfig(task="cartpole-balance-pixels",
                                         visual_randomization=True), n, dtype="float32")
    env.reset(seed=0)
    acts = torch.rand((4, n, 1), device="cuda") * 2 - 1
    for k in range(4):
        env.step(acts[k])
    T = 1000
    r = torch.randn((T, n), device="cuda")
    v = torch.randn((T, n), device="cuda")
    d = (torch.rand((T, n), device="cuda") < 0.001).float()
    b = torch.randn(n, device="cuda")
    for _ in range(2):
        P.compute_gae_batch(r, v, b, d, 0.99, 0.95)
    x = torch.randn((30 * n, 75), device="cuda")
    nz = P.DeviceRunningNormalizer(75)
    for _ in range(2):
        nz.update(x)
    torch.cuda.synchronize()
    env.check()
    print("ok")


if __name__ == "__main__":
    main()
