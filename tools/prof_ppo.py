"""Short program for ncu: two RolloutGraph phases of the PPO rollout (8192
worlds, T=30, the reference's default networks on the tensor cores)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2502_08844_b200 as dk
    from paper_2502_08844_b200 import ppo as P
    from paper_2502_08844_b200 import rollout as R

    class Cfg:
        unroll_length, reward_scaling, discounting = 30, 10.0, 0.995
        policy_obs_key = value_obs_key = "state"

    torch.manual_seed(0)
    env = dk.DeviceBatchEnv(dk.EnvConfig(task="cartpole-balance"), 8192, dtype="float32")
    obs = env.reset(seed=0)
    policy, value = R.make_policy(5, 1).cuda(), R.make_value(5).cuda()
    rg = R.RolloutGraph(env, policy, value, Cfg, obs, P.DeviceRunningNormalizer(5),
                        P.DeviceRunningNormalizer(5))
    for _ in range(2):
        rg.run()
    torch.cuda.synchronize()
    env.check()
    print("prof_ppo done")


if __name__ == "__main__":
    main()
