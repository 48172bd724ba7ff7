"""Golden outputs of ppo.evaluate (ppo.py:479-502), produced by the reference on CPU.

    python tests/golden/make_golden_evaluate.py     (needs /root/reference; CPU)

Cases: MLPPolicy on cartpole-balance (32 worlds, episode_length 25, with a policy
normaliser holding fixed statistics), the same with max_steps 10, and the CNNPolicy
on cartpole-balance-pixels (4 worlds, episode_length 6).  Two evaluations back to
back per env (the second continues the episode counters).  Saves the weights, the
normaliser and the returned dicts.
"""
import json
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

    torch.manual_seed(21)
    data, res = {}, {}
    cfg = ppo.PPOConfig(num_envs=32, unroll_length=4, num_minibatches=1, batch_size=128,
                        policy_hidden=(32, 32))
    policy = ppo.MLPPolicy(5, 1, cfg.policy_hidden)
    pn = RunningNormalizer(5)
    pn.count, pn.mean, pn.var = 100.0, np.array([0.1, 0.9, 0.0, 0.2, -0.1]), \
        np.array([0.3, 0.01, 0.05, 0.5, 2.0])
    state = ppo.TrainerState(policy=policy, value=ppo.MLPValue(5, (8,)), cfg=cfg,
                             policy_normalizer=pn)
    for k, v in policy.state_dict().items():
        data[f"mlp/{k}"] = v.numpy()
    data["pn/mean"], data["pn/var"] = pn.mean, pn.var
    env = envkit.BatchEnv(envkit.EnvConfig(task="cartpole-balance", episode_length=25, seed=5), 32)
    res["mlp"] = [ppo.evaluate(state, env), ppo.evaluate(state, env, max_steps=10)]
    pcfg = ppo.PPOConfig(num_envs=4, unroll_length=4, num_minibatches=1, batch_size=16,
                         policy_obs_key="pixels", value_obs_key="state", cnn_dense=(16,))
    cnn = ppo.CNNPolicy(3, 64, 1, dense=pcfg.cnn_dense)
    for k, v in cnn.state_dict().items():
        data[f"cnn/{k}"] = v.numpy()
    pstate = ppo.TrainerState(policy=cnn, value=ppo.MLPValue(5, (8,)), cfg=pcfg)
    penv = envkit.BatchEnv(envkit.EnvConfig(task="cartpole-balance-pixels", episode_length=6,
                                            visual_randomization=True, seed=2), 4)
    res["cnn"] = [ppo.evaluate(pstate, penv), ppo.evaluate(pstate, penv)]
    np.savez_compressed(os.path.join(OUT, "evaluate_golden.npz"), **data)
    with open(os.path.join(OUT, "evaluate_golden.json"), "w") as f:
        json.dump(res, f, indent=1)
    print(res)


if __name__ == "__main__":
    main()
