"""CPU checks of the Go1 joystick env oracle (oracle/go1env.py) -- the checker
the fused env kernel (csrc/go1env.cuh) is compared with on the GPU.

The reference has no Go1 environment, so the composition is
unpinned; these tests pin its glue against the behaviour it restates:
  * reset draws follow the Philox stream (seed, env, episode, 0) exactly, with
    every domain-randomised parameter inside its configured range;
  * a robot commanded to hold its home pose keeps standing (no termination)
    and carries its weight on its feet;
  * rewards are finite and equal the weighted sum of their 16 terms clipped
    at 0 (rewards.total_reward, rewards.py:201-211);
  * an episode truncates at episode_length, auto-resets with episode + 1 and
    reports the pre-reset observation as the terminal observation.
"""

import math

import numpy as np

from oracle import go1env as og
from oracle import oracle as orc
from paper_2502_08844_b200 import physmodel as pm


def _env(n=8, **cfg):
    base = dict(obs_noise=(0.0, 0.0, 0.0, 0.0, 0.0))
    base.update(cfg)
    return og.OracleGo1Env(pm.go1_model(), base, n)


def test_reset_draws_follow_the_stream():
    env = _env(6, seed=11)
    env.reset()
    c = env.cfg
    for i in range(6):
        w = orc.stream_raw(11, i, 0, 0, 19)
        u = (w >> np.uint64(11)).astype(np.float64) / 9007199254740992.0
        yaw = -c["yaw_range"] + 2 * c["yaw_range"] * u[0]
        np.testing.assert_allclose(env.qpos[i, 3], math.cos(0.5 * yaw), rtol=0, atol=1e-15)
        np.testing.assert_allclose(env.qpos[i, 6], math.sin(0.5 * yaw), rtol=0, atol=1e-15)
        np.testing.assert_allclose(env.qpos[i, 7:] - og.HOME,
                                   -0.1 + 0.2 * u[1:13], rtol=0, atol=1e-15)
        for k in range(3):
            assert c["cmd_lo"][k] <= env.cmd[i, k] <= c["cmd_hi"][k]
        fr, mass, kp = env.params[i]
        assert c["dr_friction"][0] <= fr <= c["dr_friction"][1]
        assert env.model.base_mass + c["dr_payload"][0] <= mass <= env.model.base_mass + c["dr_payload"][1]
        assert env.model.kp * c["dr_kp_scale"][0] <= kp <= env.model.kp * c["dr_kp_scale"][1]
    np.testing.assert_array_equal(env.qpos[:, 2], og.HOME_HEIGHT)
    np.testing.assert_array_equal(env.qvel, 0.0)


def test_home_pose_keeps_standing():
    env = _env(4, seed=3, joint_noise=0.0)
    env.reset()
    for _ in range(100):  # 2 s of simulated time
        out = env.step(np.zeros((4, 12)))
        assert not out["done"].any()
        assert np.isfinite(out["reward"]).all() and np.isfinite(out["obs"]).all()
    # settled on its feet (the PD legs give ~5 cm under the weight), at rest
    assert (np.abs(env.qpos[:, 2] - og.HOME_HEIGHT) < 0.07).all()
    assert (np.abs(env.qvel[:, :3]) < 0.02).all()


def test_reward_is_the_clipped_weighted_sum_of_terms():
    from oracle import locomotion as olo

    d = dict(zip(olo.REWARD_FIELDS, olo.REWARD_DEFAULTS))
    w = np.array([d[k] for k in ("w_lin_vel", "w_ang_vel", "w_airtime", "w_clearance", "w_phase",
                                 "w_slip", "w_orientation", "w_torque", "w_joint_pos",
                                 "w_action_rate", "w_energy", "w_pose", "w_termination",
                                 "w_standstill", "w_lin_vel_z", "w_ang_vel_xy")])
    env = _env(8, seed=5)
    env.reset()
    rng = np.random.default_rng(0)
    for _ in range(5):
        out = env.step(rng.uniform(-1, 1, (8, 12)))
        assert np.isfinite(out["terms"]).all()
        np.testing.assert_allclose(out["reward"], np.maximum(out["terms"] @ w, 0.0),
                                   rtol=1e-12, atol=1e-12)
        assert (out["reward"] >= 0).all()


def test_truncation_autoreset_and_terminal_obs():
    env = _env(3, seed=9, episode_length=4, joint_noise=0.0)
    env.reset()
    last = None
    for k in range(4):
        out = env.step(np.zeros((3, 12)))
        if k < 3:
            assert not out["trunc"].any()
            last = out
    assert out["trunc"].all() and out["terminal_mask"].all()
    np.testing.assert_array_equal(env.episode, 1)
    np.testing.assert_array_equal(env.steps, 0)
    # the terminal observation is a post-step observation of the old episode, not
    # the reset one: it differs from the new episode's first observation
    assert not np.allclose(out["terminal_obs"], out["obs"])
    assert last is not None and np.isfinite(out["terminal_obs"]).all()
