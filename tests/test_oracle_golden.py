"""Pin the CPU oracle (oracle/oracle.c) to the reference's own outputs.

The fixtures in tests/golden/envstep_golden.npz were produced by the reference
(deskrl 0.1.0) via tests/golden/make_golden.py.  The oracle restates the same
float64 arithmetic in the same order with the same libm, so everything here is
bit-exact (assert_array_equal), not a tolerance check.
"""

import numpy as np
import pytest

TASKS = ["pendulum-swingup", "cartpole-balance", "acrobot-swingup", "reacher-easy"]


def test_philox_raw_words(golden, oracle):
    for key, raw in zip(golden["philox_keys"], golden["philox_raw"]):
        seed, env, ep, step = (int(v) for v in key)
        out = oracle.stream_raw(seed, env, ep, step, 12)
        np.testing.assert_array_equal(out, raw)


def test_philox_appendix_a_kat(oracle):
    # stream_rng(0, 0, 0, 0)
    out = oracle.stream_raw(0, 0, 0, 0, 4)
    assert [hex(int(v)) for v in out] == [
        "0x2f4ba6408e4d89b", "0x3dd62b0b9ca8c5b2", "0x1c8667a55d902e79", "0x907d7a052fd5b4dc"]


@pytest.mark.parametrize("task", TASKS + ["pendulum-swingup:wide"])
def test_sample_initial(golden, oracle, task):
    keys = golden[f"reset/{task}/keys"]
    name = task.split(":")[0]
    wide = task.endswith(":wide")
    for (seed, env, ep), st, tg in zip(keys, golden[f"reset/{task}/state"],
                                       golden[f"reset/{task}/target"]):
        s, t = oracle.sample_initial(name, int(seed), int(env), int(ep), wide_init=wide)
        np.testing.assert_array_equal(s, st)
        np.testing.assert_array_equal(t, tg)


def test_cartpole_reset_appendix_a(oracle):
    s, _ = oracle.sample_initial("cartpole-balance", 0, 0, 0)
    assert tuple(s) == (-0.7815251931418695, -0.02584508034372819, -0.007771482889701236,
                        0.001288292432142674)
    s, _ = oracle.sample_initial("cartpole-balance", 7, 1023, 3)
    assert tuple(s) == (0.43868601084788317, 0.03524527976706099, 0.00935161601640694,
                        0.0024283818296617216)


@pytest.mark.parametrize("task", TASKS)
def test_step_reward_obs(golden, oracle, task):
    g = {k: golden[f"step/{task}/{k}"] for k in ("s", "a", "target", "ns", "r", "info", "obs")}
    for i in range(len(g["s"])):
        ns = oracle.step_dynamics(task, g["s"][i], g["a"][i])
        np.testing.assert_array_equal(ns, g["ns"][i])
        tgt = g["target"][i] if task == "reacher-easy" else None
        r, info = oracle.reward(task, ns, tgt)
        assert r == g["r"][i]
        np.testing.assert_array_equal(info, g["info"][i])
        np.testing.assert_array_equal(oracle.state_obs(task, ns, tgt), g["obs"][i])


def test_tol(golden, oracle):
    for x, lo, hi, m, want in golden["tol"]:
        assert oracle.tol(x, lo, hi, m) == want
    assert oracle.tol(1.2, -0.25, 0.25, 1.55) == 0.42106547754029083


def _traj_names(golden):
    return sorted({k.split("/")[1] for k in golden.files if k.startswith("traj/")})


def test_batch_trajectories(golden, oracle):
    from oracle.oracle import OracleBatchEnv

    class _P:  # the "damped" DynamicsParams override used by make_golden.py
        pass

    names = _traj_names(golden)
    assert len(names) >= 6
    for name in names:
        g = lambda k: golden[f"traj/{name}/{k}"]  # noqa: E731
        dt = float(g("meta_dt"))
        params = None
        if str(g("meta_params")) == "damped":
            import oracle.oracle as orc

            params = _P()
            for f, v in zip(orc.PARAM_FIELDS, orc.PARAM_DEFAULTS):
                setattr(params, f, v)
            params.link_damping, params.link2_mass, params.elbow_torque_limit = 0.1, 1.3, 6.0
        env = OracleBatchEnv(str(g("meta_task")), int(g("meta_n")),
                             episode_length=int(g("meta_ep_len")),
                             action_repeat=int(g("meta_rep")), wide_init=bool(g("meta_wide")),
                             dt=None if dt < 0 else dt, params=params)
        obs0 = env.reset(seed=int(g("meta_seed")))
        np.testing.assert_array_equal(obs0, g("obs0"))
        acts = g("acts")
        for k in range(acts.shape[0]):
            if k == int(g("mid_reset_step")):
                np.testing.assert_array_equal(env.reset(), g("obs_mid_reset"))
            obs, rew, done, trunc, term, mask, info = env.step(acts[k])
            np.testing.assert_array_equal(obs, g("obs")[k], err_msg=f"{name} step {k}")
            np.testing.assert_array_equal(obs, g("priv")[k])
            np.testing.assert_array_equal(rew, g("rew")[k])
            np.testing.assert_array_equal(done, g("done")[k])
            np.testing.assert_array_equal(trunc, g("trunc")[k])
            np.testing.assert_array_equal(mask, g("term_mask")[k])
            np.testing.assert_array_equal(term[mask], g("term_obs")[k][mask])
            np.testing.assert_array_equal(info, g("info")[k])
        np.testing.assert_array_equal(env.state, g("final_state"))
        np.testing.assert_array_equal(env.steps, g("final_steps"))
        np.testing.assert_array_equal(env.episode, g("final_episode"))


def test_long_horizon_bit_exact(golden, oracle):
    from oracle.oracle import OracleBatchEnv

    n, steps = int(golden["long/n"]), int(golden["long/steps"])
    env = OracleBatchEnv("cartpole-balance", n, episode_length=400)
    env.reset(seed=77)
    acts = np.random.default_rng(int(golden["long/acts_seed"])).uniform(-1, 1, (steps, n, 1))
    obs, rew, done, trunc, *_ = env.rollout(acts, nthreads=2)
    np.testing.assert_array_equal(obs[-1], golden["long/final_obs"])
    np.testing.assert_array_equal(rew.sum(0), golden["long/rsum"])
    np.testing.assert_array_equal(trunc.sum(0), golden["long/ntrunc"])
    np.testing.assert_array_equal(env.state, golden["long/final_state"])


def test_oracle_error_semantics(golden, oracle):
    from oracle.oracle import OracleBatchEnv, OracleError

    env = OracleBatchEnv("cartpole-balance", 4, episode_length=2)
    with pytest.raises(OracleError) as e:
        env.step(np.zeros((4, 1)))
    assert e.value.code == 1 and e.value.index == 0
    env.reset(seed=0)
    a = np.zeros((4, 1))
    a[2, 0] = np.nan
    with pytest.raises(OracleError) as e:
        env.step(a)
    assert e.value.code == 2 and e.value.index == 2
