"""Golden vectors for the on-device rollout (ppo.collect_rollout, ppo.py:295-378),
produced by the reference itself on CPU.

    python tests/golden/make_golden_rollout.py     (needs /root/reference; CPU)

rollout_golden_default.npz: the same with the default network sizes.
A 64-world cartpole BatchEnv with episode_length 5 (truncation bootstraps inside
the 8-step unroll), the reference's MLPPolicy / MLPValue (small hidden sizes),
observation normalisers, two collect_rollout phases.  Saves the network
weights, the policy noise the reference's generator drew (torch.randn per
step), every RolloutBatch field, the resume observation, the mean raw reward
and the normaliser statistics after each phase.
"""
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def main(policy_hidden=(32, 32), value_hidden=(48, 48), out_name="rollout_golden.npz"):
    sys.path.insert(0, REF)
    import torch
    from deskrl import envkit, ppo
    from deskrl.mathcore import RunningNormalizer

    torch.manual_seed(5)
    N, T = 64, 8
    cfg = ppo.PPOConfig(num_envs=N, unroll_length=T, num_minibatches=4, batch_size=128,
                        policy_hidden=policy_hidden,
                        value_hidden=value_hidden, reward_scaling=10.0, discounting=0.995)
    env = envkit.BatchEnv(envkit.EnvConfig(task="cartpole-balance", episode_length=5), N)
    obs = env.reset(seed=3)
    policy = ppo.MLPPolicy(5, 1, cfg.policy_hidden)
    value = ppo.MLPValue(5, cfg.value_hidden)
    state = ppo.TrainerState(policy=policy, value=value, cfg=cfg,
                             policy_normalizer=RunningNormalizer(5),
                             value_normalizer=RunningNormalizer(5))
    data = {"obs0": obs["state"]}
    for k, v in list(policy.state_dict().items()):
        data[f"policy/{k}"] = v.numpy()
    for k, v in list(value.state_dict().items()):
        data[f"value/{k}"] = v.numpy()
    seed = 17
    g_noise = torch.Generator()
    g_noise.manual_seed(seed)
    g = torch.Generator()
    g.manual_seed(seed)
    for phase in range(2):
        data[f"p{phase}/noise"] = np.stack(
            [torch.randn((N, 1), generator=g_noise).numpy() for _ in range(T)])
        batch, obs, mean_r = ppo.collect_rollout(env, state, obs, g)
        for f in ("policy_obs", "value_obs", "actions", "pre_tanh", "log_probs", "rewards",
                  "dones", "values", "bootstrap"):
            data[f"p{phase}/{f}"] = getattr(batch, f)
        data[f"p{phase}/next_obs"] = obs["state"]
        data[f"p{phase}/mean_reward"] = np.array(mean_r)
        for name, nz in (("pn", state.policy_normalizer), ("vn", state.value_normalizer)):
            data[f"p{phase}/{name}_count"] = np.array(nz.count)
            data[f"p{phase}/{name}_mean"] = nz.mean
            data[f"p{phase}/{name}_var"] = nz.var
    path = os.path.join(OUT, out_name)
    np.savez_compressed(path, **data)
    print(f"wrote {path} ({os.path.getsize(path)} bytes, {len(data)} arrays)")


if __name__ == "__main__":
    main()
    # the reference's default network sizes (PPOConfig: policy 4 x 128, value
    # 5 x 256): the shapes the tensor-core MLP kernel serves
    main((128, 128, 128, 128), (256, 256, 256, 256, 256), "rollout_golden_default.npz")
