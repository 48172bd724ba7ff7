"""Golden data for the wire / on-disk formats, produced by
the reference:

* serve.serve_stdio replies to a scripted session (state and pixel envs,
  errors) -> tests/golden/serve_session.jsonl (request / reply pairs);
* ppo.save_checkpoint of a small TrainerState with normalisers ->
  tests/golden/ref_checkpoint.bin (+ the weights / stats it holds in
  tests/golden/ref_checkpoint.npz).

    python tests/golden/make_golden_formats.py     (needs /root/reference; CPU)
"""
import io
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def session():
    rng = np.random.default_rng(9)
    reqs = [{"op": "version"},
            {"op": "make_env", "task": "cartpole-balance",
             "config": {"num_envs": 3, "seed": 5, "episode_length": 4}},
            {"op": "reset", "handle": 1, "seed": 5}]
    for _ in range(6):
        reqs.append({"op": "step", "handle": 1,
                     "actions": rng.uniform(-1, 1, (3, 1)).tolist()})
    reqs += [{"op": "step", "handle": 1, "actions": [[0.1, 0.2]]},
             {"op": "step", "handle": 7, "actions": [[0.0]]},
             {"op": "make_env", "task": "cartpole-balance", "config": {"bogus": 1}},
             {"op": "make_env", "task": "pendulum-swingup", "config": {"num_envs": 2}},
             {"op": "reset", "handle": 2},
             {"op": "step", "handle": 2, "actions": [[0.5], [-0.25]]},
             {"op": "make_env", "task": "cartpole-balance-pixels",
              "config": {"num_envs": 2, "image_size": 16, "visual_randomization": True,
                         "seed": 3}},
             {"op": "reset", "handle": 3, "seed": 3},
             {"op": "step", "handle": 3, "actions": [[0.3], [-0.7]]},
             {"op": "nope"},
             {"op": "close", "handle": 1}, {"op": "close", "handle": 2},
             {"op": "close", "handle": 3}, {"op": "close", "handle": 1}]
    return reqs


def main():
    sys.path.insert(0, REF)
    import torch
    from deskrl import ppo, serve
    from deskrl.mathcore import RunningNormalizer

    reqs = session()
    out = io.StringIO()
    serve.serve_stdio(io.StringIO("\n".join(json.dumps(r) for r in reqs) + "\n"), out)
    replies = out.getvalue().strip().split("\n")
    assert len(replies) == len(reqs)
    with open(os.path.join(OUT, "serve_session.jsonl"), "w") as f:
        for q, r in zip(reqs, replies):
            f.write(json.dumps({"request": q, "reply": json.loads(r)}) + "\n")

    torch.manual_seed(3)
    cfg = ppo.PPOConfig(num_envs=8, unroll_length=4, num_minibatches=2, batch_size=16,
                        policy_hidden=(8, 8), value_hidden=(6,))
    st = ppo.TrainerState(policy=ppo.MLPPolicy(5, 1, (8, 8)), value=ppo.MLPValue(5, (6,)),
                          cfg=cfg,
                          policy_normalizer=RunningNormalizer(5, 40.0, np.arange(5) * 0.1,
                                                              np.arange(5) + 0.5),
                          value_normalizer=RunningNormalizer(5, 12.0, -np.arange(5) * 0.3,
                                                             np.arange(5) * 2 + 0.25))
    path = os.path.join(OUT, "ref_checkpoint.bin")
    ppo.save_checkpoint(st, path, extra={"env_steps": 1234, "note": "golden"})
    arrays = {f"policy/{k}": v.numpy() for k, v in st.policy.state_dict().items()}
    arrays.update({f"value/{k}": v.numpy() for k, v in st.value.state_dict().items()})
    for key, n in (("pn", st.policy_normalizer), ("vn", st.value_normalizer)):
        arrays[f"{key}/count"] = np.array(n.count)
        arrays[f"{key}/mean"] = n.mean
        arrays[f"{key}/var"] = n.var
    arrays["config_hash"] = np.array(cfg.config_hash())
    np.savez(os.path.join(OUT, "ref_checkpoint.npz"), **arrays)
    print("wrote serve_session.jsonl, ref_checkpoint.bin/.npz")


if __name__ == "__main__":
    main()
