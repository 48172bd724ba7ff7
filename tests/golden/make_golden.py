"""Generate the golden fixtures for the env step from the REFERENCE itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports deskrl 0.1.0 from /root/reference/pkg/src and records, for fixed
seeds, the reference's outputs for every function on the hot path (SURVEY.md
§8a rows A1-A12): Philox stream words (envkit.py:41-49), initial-state
sampling (envkit.py:262-272, 302-309, 387-390, 418-424), the scalar task
step/reward/obs (envkit.py:274-453), ``_tol`` (envkit.py:216-221), and whole
BatchEnv trajectories with autoreset / action_repeat / dt overrides
(envkit.py:502-552, 616-646), plus the error behaviour.  The fixtures are
committed; nothing on the GPU box reads /root/reference.
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))

TASKS = ["pendulum-swingup", "cartpole-balance", "acrobot-swingup", "reacher-easy"]


def _import_ref():
    sys.path.insert(0, REF)
    import deskrl  # noqa: F401
    from deskrl import dynamics, envkit, mathcore, randomization

    return envkit, dynamics, mathcore, randomization


def philox_cases(envkit):
    keys = np.array(
        [
            [0, 0, 0, 0],
            [0, 1, 0, 0],
            [7, 1023, 3, 0],
            [123456789, 5, 2**32 + 9, 0],  # episode wraps mod 2^32 in the key
            [2**63 + 11, 4095, 17, 0],
            [42, 8191, 999, 5],           # nonzero counter start
        ],
        dtype=object,
    )
    raw = []
    for seed, env, ep, step in keys:
        g = envkit.stream_rng(int(seed), int(env), int(ep), int(step))
        raw.append(g.bit_generator.random_raw(12))
    return np.array(keys.tolist(), dtype=np.uint64), np.array(raw, dtype=np.uint64)


def reset_cases(envkit, dynamics):
    rng = np.random.default_rng(1)
    out = {}
    for task in TASKS + ["pendulum-swingup:wide"]:
        name, wide = (task.split(":")[0], True) if ":" in task else (task, False)
        cls = envkit._TASKS[name]
        t = cls(dynamics.DynamicsParams())
        t.wide_init = wide
        keys = np.stack(
            [rng.integers(0, 2**40, 64), rng.integers(0, 100000, 64), rng.integers(0, 5000, 64)],
            axis=1,
        ).astype(np.int64)
        states, targets = [], []
        for seed, env, ep in keys:
            s = t.sample_initial(envkit.stream_rng(int(seed), int(env), int(ep), 0))
            if len(s) == 2 and isinstance(s[1], np.ndarray):
                states.append(list(s[0]))
                targets.append(list(s[1]))
            else:
                states.append(list(s) + [0.0] * (4 - len(s)))
                targets.append([0.0, 0.0])
        out[task] = (keys, np.array(states), np.array(targets))
    return out


def _random_states(task, rng, m):
    if task == "pendulum-swingup":
        s = np.stack([rng.uniform(-40, 40, m), rng.uniform(-30, 30, m), 0 * np.ones(m),
                      0 * np.ones(m)], 1)
    elif task == "cartpole-balance":
        s = np.stack([rng.uniform(-1.85, 1.85, m), rng.uniform(-60, 60, m),
                      rng.uniform(-8, 8, m), rng.uniform(-30, 30, m)], 1)
        s[:8, 0] = [1.8, -1.8, 1.799, -1.799, 1.7999999, -1.7999999, 0.0, 0.25]
        s[:8, 2] = [3.0, -3.0, 5.0, -5.0, 0.1, -0.1, 0.0, 0.0]
    else:
        s = np.stack([rng.uniform(-12, 12, m), rng.uniform(-12, 12, m), rng.uniform(-15, 15, m),
                      rng.uniform(-15, 15, m)], 1)
    return s


def step_cases(envkit, dynamics):
    """Scalar step_dynamics -> reward -> state_obs for random states/actions."""
    rng = np.random.default_rng(2)
    out = {}
    for task in TASKS:
        cls = envkit._TASKS[task]
        t = cls(dynamics.DynamicsParams().with_dt(cls.default_dt))
        m = 512
        s = _random_states(task, rng, m)
        a = rng.uniform(-1.6, 1.6, (m, cls.action_dim))
        a[:4] = [[1.0] * cls.action_dim, [-1.0] * cls.action_dim, [0.0] * cls.action_dim,
                 [1e-300] * cls.action_dim]
        target = np.stack([rng.uniform(-1.9, 1.9, m), rng.uniform(-1.9, 1.9, m)], 1)
        ns, r, info, obs = [], [], [], []
        for i in range(m):
            st = tuple(float(v) for v in s[i, : cls.state_dim])
            nxt = t.step_dynamics(st, tuple(float(v) for v in a[i]))
            if task == "reacher-easy":
                rr, inf = t.reward(nxt, None, target[i])
                ob = t.state_obs(nxt, target[i])
            else:
                rr, inf = t.reward(nxt, None)
                ob = t.state_obs(nxt)
            ns.append(list(nxt) + [0.0] * (4 - len(nxt)))
            r.append(rr)
            info.append(list(inf.values()))
            obs.append(ob)
        out[task] = dict(s=s, a=a, target=target, ns=np.array(ns), r=np.array(r),
                         info=np.array(info), obs=np.array(obs))
    return out


def tol_cases(envkit):
    rng = np.random.default_rng(3)
    rows = []
    for _ in range(2000):
        lo = rng.uniform(-2, 2)
        hi = lo + abs(rng.normal(0, 1)) * (rng.uniform() < 0.8)
        margin = rng.uniform(0.05, 6)
        x = rng.uniform(lo - 3 * margin, hi + 3 * margin)
        rows.append([x, lo, hi, margin, envkit._tol(x, lo, hi, margin)])
    rows.append([1.2, -0.25, 0.25, 1.55, envkit._tol(1.2, -0.25, 0.25, 1.55)])
    rows.append([1.8, -0.25, 0.25, 1.55, envkit._tol(1.8, -0.25, 0.25, 1.55)])
    rows.append([0.25, -0.25, 0.25, 1.55, envkit._tol(0.25, -0.25, 0.25, 1.55)])
    return np.array(rows)


TRAJ_CASES = [
    # name, task, num_envs, steps, episode_length, action_repeat, dt, seed, wide, params
    ("cartpole", "cartpole-balance", 48, 60, 13, 1, None, 0, False, None),
    ("cartpole_rep3", "cartpole-balance", 32, 30, 7, 3, None, 5, False, None),
    ("pendulum_wide", "pendulum-swingup", 32, 40, 11, 2, None, 3, True, None),
    ("pendulum", "pendulum-swingup", 32, 30, 1000, 1, 0.02, 9, False, None),
    ("acrobot", "acrobot-swingup", 32, 40, 9, 1, None, 4, False, "damped"),
    ("reacher", "reacher-easy", 32, 40, 10, 2, None, 11, False, None),
]


def trajectory_cases(envkit, dynamics):
    out = {}
    for name, task, n, steps, ep_len, rep, dt, seed, wide, params in TRAJ_CASES:
        p = None
        if params == "damped":
            p = dynamics.DynamicsParams(link_damping=0.1, link2_mass=1.3, elbow_torque_limit=6.0)
        cfg = envkit.EnvConfig(task=task, episode_length=ep_len, action_repeat=rep, dt=dt,
                               wide_init=wide)
        env = envkit.BatchEnv(cfg, n, params=p)
        rng = np.random.default_rng(100 + seed)
        obs0 = env.reset(seed=seed)
        A = env.action_dim
        acts = rng.uniform(-1.3, 1.3, (steps, n, A))
        O = obs0["state"].shape[1]
        rec = dict(
            obs0=obs0["state"], acts=acts,
            obs=np.zeros((steps, n, O)), priv=np.zeros((steps, n, O)), rew=np.zeros((steps, n)),
            done=np.zeros((steps, n), bool), trunc=np.zeros((steps, n), bool),
            term_mask=np.zeros((steps, n), bool), term_obs=np.zeros((steps, n, O)),
            info=None,
        )
        infos_all = []
        for k in range(steps):
            if k == steps // 2:
                # reset() without a seed continues the episode counters (envkit.py:616-623)
                rec["obs_mid_reset"] = env.reset()["state"]
                rec["mid_reset_step"] = np.int64(k)
            o, r, d, tr, infos = env.step(acts[k])
            rec["obs"][k] = o["state"]
            rec["priv"][k] = o["privileged_state"]
            rec["rew"][k] = r
            rec["done"][k] = d
            rec["trunc"][k] = tr
            keys = [kk for kk in infos[0] if kk != "terminal_observation"]
            infos_all.append([[inf[kk] for kk in keys] for inf in infos])
            for i, inf in enumerate(infos):
                if "terminal_observation" in inf:
                    rec["term_mask"][k, i] = True
                    rec["term_obs"][k, i] = inf["terminal_observation"]["state"]
        rec["info"] = np.array(infos_all)
        rec["final_state"] = np.array([list(e.state) + [0.0] * (4 - len(e.state))
                                       for e in env.envs])
        rec["final_steps"] = np.array([e.steps for e in env.envs], dtype=np.int64)
        rec["final_episode"] = np.array([e._episode for e in env.envs], dtype=np.int64)
        meta = dict(task=task, n=n, steps=steps, ep_len=ep_len, rep=rep,
                    dt=-1.0 if dt is None else dt, seed=seed, wide=wide,
                    params="" if params is None else params)
        out[name] = (rec, meta)
    return out


def long_horizon_case(envkit):
    """Cartpole, 256 worlds x 1000 steps, episode_length 400: final state and
    per-world reward sums (checks the oracle stays bit-exact through chaos and
    autoresets without storing the whole trajectory)."""
    n, steps = 256, 1000
    env = envkit.BatchEnv(envkit.EnvConfig(task="cartpole-balance", episode_length=400), n)
    env.reset(seed=77)
    rng = np.random.default_rng(77)
    acts = rng.uniform(-1, 1, (steps, n, 1))
    rsum = np.zeros(n)
    ntrunc = np.zeros(n, dtype=np.int64)
    for k in range(steps):
        o, r, d, tr, infos = env.step(acts[k])
        rsum += r
        ntrunc += tr
    return dict(acts_seed=np.int64(77), n=np.int64(n), steps=np.int64(steps),
                final_obs=o["state"], rsum=rsum, ntrunc=ntrunc,
                final_state=np.array([list(e.state) for e in env.envs]))


def error_cases(envkit, mathcore, randomization):
    res = {}
    env = envkit.BatchEnv(envkit.EnvConfig(task="cartpole-balance", episode_length=3), 4)
    try:
        env.envs[0].step([0.0])
    except envkit.UsageError as e:
        res["step_before_reset"] = ("UsageError", str(e))
    env.reset(seed=0)
    a = np.zeros((4, 1))
    a[2, 0] = np.nan
    try:
        env.step(a)
    except mathcore.InvalidInputError as e:
        res["nan_action"] = ("InvalidInputError", str(e))
    try:
        env.step(np.zeros((3, 1)))
    except mathcore.InvalidInputError as e:
        res["batch_mismatch"] = ("InvalidInputError", str(e))
    try:
        envkit.BatchEnv(envkit.EnvConfig(task="go1-joystick"), 2)
    except randomization.ConfigError as e:
        res["unknown_task"] = ("ConfigError", str(e))
    env2 = envkit.BatchEnv(envkit.EnvConfig(task="cartpole-balance", episode_length=2), 2)
    env2.reset(seed=1)
    env2.step(np.zeros((2, 1)), autoreset=False)
    env2.step(np.zeros((2, 1)), autoreset=False)
    try:
        env2.step(np.zeros((2, 1)), autoreset=False)
    except envkit.UsageError as e:
        res["step_after_trunc_no_autoreset"] = ("UsageError", str(e))
    res["registered_tasks"] = ("list", ",".join(envkit.registered_tasks()))
    return res


def main():
    envkit, dynamics, mathcore, randomization = _import_ref()
    data = {}
    k, raw = philox_cases(envkit)
    data["philox_keys"] = k
    data["philox_raw"] = raw
    for task, (keys, st, tg) in reset_cases(envkit, dynamics).items():
        data[f"reset/{task}/keys"] = keys
        data[f"reset/{task}/state"] = st
        data[f"reset/{task}/target"] = tg
    for task, d in step_cases(envkit, dynamics).items():
        for key, v in d.items():
            data[f"step/{task}/{key}"] = v
    data["tol"] = tol_cases(envkit)
    for name, (rec, meta) in trajectory_cases(envkit, dynamics).items():
        for key, v in rec.items():
            data[f"traj/{name}/{key}"] = v
        for key, v in meta.items():
            data[f"traj/{name}/meta_{key}"] = np.array(v)
    for key, v in long_horizon_case(envkit).items():
        data[f"long/{key}"] = v
    for key, (kind, msg) in error_cases(envkit, mathcore, randomization).items():
        data[f"err/{key}"] = np.array([kind, msg])
    path = os.path.join(OUT, "envstep_golden.npz")
    np.savez_compressed(path, **data)
    print(f"wrote {path} ({os.path.getsize(path)} bytes, {len(data)} arrays)")


if __name__ == "__main__":
    main()
