"""Golden vectors for the on-device pixel-policy rollout: ppo.collect_rollout
(ppo.py:295-378) with the reference's CNNPolicy on pixel_normalize'd stacks
(_prep_policy_obs, ppo.py:278-285) and an MLP value on the state, produced by the
reference itself on CPU.

    python tests/golden/make_golden_rollout_pixels.py     (needs /root/reference; CPU)

4 cartpole-balance-pixels worlds with visual randomisation, episode_length 4
(truncation bootstraps inside the 6-step unroll), a value normaliser (the
reference gives pixel policies none).  Saves the weights, the noise, every
RolloutBatch field (policy observations: first and last step in full, per-(t, n, c)
sums for all steps), the resume observation and the value-normaliser statistics.
"""
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF)
    import torch
    from deskrl import envkit, ppo
    from deskrl.mathcore import RunningNormalizer

    torch.manual_seed(11)
    N, T = 4, 6
    cfg = ppo.PPOConfig(num_envs=N, unroll_length=T, num_minibatches=2, batch_size=12,
                        policy_obs_key="pixels", value_obs_key="state", cnn_dense=(32,),
                        value_hidden=(48, 48), reward_scaling=10.0, discounting=0.995)
    env = envkit.BatchEnv(envkit.EnvConfig(task="cartpole-balance-pixels", episode_length=4,
                                           visual_randomization=True), N)
    obs = env.reset(seed=6)
    policy = ppo.CNNPolicy(3, 64, 1, dense=cfg.cnn_dense)
    value = ppo.MLPValue(5, cfg.value_hidden)
    state = ppo.TrainerState(policy=policy, value=value, cfg=cfg,
                             value_normalizer=RunningNormalizer(5))
    data = {"obs0": obs["state"]}
    for k, v in list(policy.state_dict().items()):
        data[f"policy/{k}"] = v.numpy()
    for k, v in list(value.state_dict().items()):
        data[f"value/{k}"] = v.numpy()
    g_noise = torch.Generator()
    g_noise.manual_seed(23)
    g = torch.Generator()
    g.manual_seed(23)
    data["noise"] = np.stack([torch.randn((N, 1), generator=g_noise).numpy() for _ in range(T)])
    batch, obs, mean_r = ppo.collect_rollout(env, state, obs, g)
    po = batch.policy_obs
    data["policy_obs_first"] = po[0]
    data["policy_obs_last"] = po[-1]
    data["policy_obs_sums"] = po.astype(np.float64).sum(axis=(3, 4))
    for f in ("value_obs", "actions", "pre_tanh", "log_probs", "rewards", "dones", "values",
              "bootstrap"):
        data[f] = getattr(batch, f)
    data["next_obs"] = obs["state"]
    data["mean_reward"] = np.array(mean_r)
    nz = state.value_normalizer
    data["vn_count"], data["vn_mean"], data["vn_var"] = np.array(nz.count), nz.mean, nz.var
    path = os.path.join(OUT, "rollout_pixels_golden.npz")
    np.savez_compressed(path, **data)
    print(f"wrote {path} ({os.path.getsize(path)} bytes, {len(data)} arrays)")


if __name__ == "__main__":
    main()
