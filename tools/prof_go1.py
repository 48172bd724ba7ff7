"""Short program for ncu: the fused Go1 env kernel and the physics kernel at
8192 worlds (f32), a few launches each.

    ncu ... -k regex:go1_env_kernel python tools/prof_go1.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from oracle import physics as op
    from paper_2502_08844_b200 import go1env as G
    from paper_2502_08844_b200 import physics as P
    from paper_2502_08844_b200 import physmodel as pm

    n, K = 8192, int(os.environ.get("PROF_K", "10"))
    dt = os.environ.get("PROF_DTYPE", "float32")
    env = G.DeviceGo1Env(n, G.Go1Config(), dtype=dt)
    env.reset(seed=0)
    acts = torch.rand((K, n, 12), device="cuda", dtype=env.dtype) * 2 - 1
    out = env.outputs(K)
    for _ in range(3):
        env.rollout(acts, out=out)
    env.check()
    sim = P.DevicePhysics(pm.go1_model(), n, dtype=dt)
    q, v, c = op.random_states(n, seed=1)
    t = lambda x: torch.as_tensor(x, device="cuda", dtype=sim.dtype)  # noqa: E731
    sim.set_state(t(q), t(v))
    for _ in range(3):
        sim.step(t(c), 5 * K, diag=False)
    sim.check()
    torch.cuda.synchronize()
    print("prof_go1 done")


if __name__ == "__main__":
    main()
