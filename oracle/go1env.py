"""Go1 joystick env oracle: the fused kernel's control step (csrc/go1env.cuh)
composed from the repo's independent oracles, in float64.

TEST INFRASTRUCTURE ONLY (see oracle/oracle.py).  UNPINNED: the reference has
no Go1 environment.  The pieces it composes are:
  * physics: oracle/physics.c (G1-G4; pinned by physics KATs);
  * reward and observation: oracle/locomotion.c, pinned bit-exact against
    the reference's rewards.total_reward / build_locomotion_observation
    (tests/test_oracle_loco.py);
  * gait bookkeeping: mathcore.wrap_angle / advance_phase (mathcore.py:143-171),
    rewards.swing_height_profile (rewards.py:92-94), envkit.action_to_target
    absolute mode (envkit.py:111-131), restated here in NumPy;
  * Philox reset draws: oracle.stream_raw + NumPy's Generator.uniform formula.
The glue follows include/deskrl_b200.h "Go1 joystick environment".
"""

from __future__ import annotations

import math

import numpy as np

from . import locomotion as olo
from . import oracle as orc
from . import physics as op

HOME = np.tile([0.0, 0.9, -1.8], 4)
PHASE0 = np.array([0.0, math.pi, math.pi, 0.0])
HOME_HEIGHT = 0.278
TWO_PI = 2.0 * math.pi


def default_config():
    return dict(episode_length=1000, ctrl_dt=0.02, action_scale=0.5, gait_freq=1.5,
                term_height=0.12, cmd_lo=(-1.5, -0.8, -1.2), cmd_hi=(1.5, 0.8, 1.2),
                joint_noise=0.1, yaw_range=math.pi, obs_noise=(0.05, 0.1, 0.2, 0.01, 1.5),
                seed=0, reward={}, dr_friction=(0.4, 1.0), dr_payload=(-0.5, 1.5),
                dr_kp_scale=(0.9, 1.1))


def _uniform(words, lo, hi):
    return lo + (hi - lo) * ((words >> np.uint64(11)).astype(np.float64) / 9007199254740992.0)


def wrap_angle(phi):
    return np.mod(phi + math.pi, TWO_PI) - math.pi


class OracleGo1Env:
    def __init__(self, model, cfg, num_worlds, env_index_offset=0):
        self.model, self.mc = model, model.to_c()
        self.cfg = {**default_config(), **cfg}
        self.n = num_worlds
        self.env0 = env_index_offset
        self.substeps = int(round(self.cfg["ctrl_dt"] / model.timestep))
        n = num_worlds
        self.qpos, self.qvel = np.zeros((n, 19)), np.zeros((n, 18))
        self.cmd, self.phase, self.air = np.zeros((n, 3)), np.zeros((n, 4)), np.zeros((n, 4))
        self.last_contact = np.zeros((n, 4), bool)
        self.prev = np.zeros((n, 12))
        self.params = np.zeros((n, 3))  # friction, trunk mass, kp (this episode's draw)
        self.steps = np.zeros(n, np.int64)
        self.episode = np.zeros(n, np.int64)

    # -- pieces
    def _reset_world(self, i):
        c = self.cfg
        w = orc.stream_raw(c["seed"], self.env0 + i, int(self.episode[i]), 0, 19)
        yaw = _uniform(w[0:1], -c["yaw_range"], c["yaw_range"])[0]
        jn = _uniform(w[1:13], -c["joint_noise"], c["joint_noise"])
        cmd = [_uniform(w[13 + k:14 + k], c["cmd_lo"][k], c["cmd_hi"][k])[0] for k in range(3)]
        # randomize_params kinds (randomization.py:156-181): friction replaced,
        # payload added to the trunk mass, kp scaled
        dr = [_uniform(w[16 + k:17 + k], *c[f])[0]
              for k, f in enumerate(("dr_friction", "dr_payload", "dr_kp_scale"))]
        self.params[i] = (dr[0], self.model.base_mass + dr[1], self.model.kp * dr[2])
        q = np.zeros(19)
        q[2] = HOME_HEIGHT
        q[3], q[6] = math.cos(0.5 * yaw), math.sin(0.5 * yaw)
        q[7:] = HOME + jn
        self.qpos[i], self.qvel[i] = q, 0.0
        self.cmd[i] = cmd
        self.phase[i] = PHASE0
        self.air[i] = 0.0
        self.prev[i] = 0.0
        self.steps[i] = 0

    def _frame(self, i, act, tau, reset_frame, done=False):
        """The LocomotionFrame of world i (and the contact flags)."""
        c, m = self.cfg, self.model
        fp, fv = op.foot_kin(self.mc, self.qpos[i:i + 1], self.qvel[i:i + 1])
        fp, fv = fp[0], fv[0]
        contact = fp[:, 2] - m.foot_radius < 0
        if not reset_frame:
            self.air[i] = self.air[i] + c["ctrl_dt"]
            self.phase[i] = wrap_angle(self.phase[i] + TWO_PI * c["gait_freq"] * c["ctrl_dt"])
        td = np.zeros(4, bool) if reset_frame else (contact & ~self.last_contact[i])
        q = self.qpos[i]
        w_, x, y, z = q[3:7]
        R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w_ * z), 2 * (x * z + w_ * y)],
                      [2 * (x * y + w_ * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w_ * x)],
                      [2 * (x * z - w_ * y), 2 * (y * z + w_ * x), 1 - 2 * (x * x + y * y)]])
        sh = self.cfg["reward"].get("swing_height", 0.08)
        fr = {"base_orientation": q[3:7][None], "base_lin_vel": (R.T @ self.qvel[i, :3])[None],
              "base_ang_vel": self.qvel[i, 3:6][None], "joint_pos": q[7:][None],
              "joint_vel": self.qvel[i, 6:][None], "joint_torque": np.asarray(tau)[None],
              "foot_height": (fp[:, 2] - m.foot_radius)[None],
              "foot_height_des": (sh * np.maximum(0.0, np.sin(self.phase[i])))[None],
              "foot_vel_xy": fv[:, :2].reshape(1, 8).reshape(1, 4, 2),
              "foot_contact": contact[None], "airtime": self.air[i][None],
              "touchdown": td[None], "phase": self.phase[i][None], "command": self.cmd[i][None],
              "action": np.asarray(act)[None], "prev_action": self.prev[i][None],
              "joint_nominal": HOME, "joint_default": HOME, "done": np.array([done])}
        return fr, contact, R

    def _obs(self, i, fr, act):
        c = self.cfg
        noise = list(c["obs_noise"]) if any(v > 0 for v in c["obs_noise"]) else None
        st, pr, bad = olo.loco_obs(fr, np.asarray(act)[None], self.cmd[i][None], noise,
                                   (c["seed"], self.env0 + i, int(self.episode[i]),
                                    int(self.steps[i]) + 1))
        assert bad == -1
        return st[0], pr[0]

    # -- API
    def reset(self, seed=None):
        if seed is not None:
            self.cfg["seed"] = int(seed)
        n = self.n
        obs, priv = np.zeros((n, 56)), np.zeros((n, 75))
        for i in range(n):
            self.episode[i] = 0
            self._reset_world(i)
            fr, contact, _ = self._frame(i, np.zeros(12), np.zeros(12), True)
            self.last_contact[i] = contact
            obs[i], priv[i] = self._obs(i, fr, np.zeros(12))
        return obs, priv

    def step(self, actions):
        c, n = self.cfg, self.n
        out = {"obs": np.zeros((n, 56)), "priv": np.zeros((n, 75)), "reward": np.zeros(n),
               "done": np.zeros(n, bool), "trunc": np.zeros(n, bool), "terms": np.zeros((n, 16)),
               "terminal_obs": np.zeros((n, 56)), "terminal_mask": np.zeros(n, bool)}
        a = np.clip(np.nan_to_num(np.asarray(actions, np.float64), nan=0.0), -1.0, 1.0)
        ctrl = HOME + c["action_scale"] * a
        # physics per world with the world's own randomised model
        ph = {"act_force": np.zeros((n, 12))}
        for i in range(n):
            m = self.model.to_c()
            m.friction, m.base_mass, m.kp = self.params[i]
            r = op.step(m, self.qpos[i:i + 1], self.qvel[i:i + 1], ctrl[i:i + 1], self.substeps)
            self.qpos[i], self.qvel[i] = r["qpos"][0], r["qvel"][0]
            ph["act_force"][i] = r["act_force"][0]
        for i in range(n):
            fr, contact, R = self._frame(i, a[i], ph["act_force"][i], False)
            done = bool(R[2, 2] < 0 or self.qpos[i, 2] < c["term_height"])
            fr["done"] = np.array([done])
            self.steps[i] += 1
            trunc = bool(self.steps[i] >= c["episode_length"])
            terms, unc, tot, bad = olo.total_reward(fr, **c["reward"])
            st, pr = self._obs(i, fr, a[i])
            self.air[i] = np.where(contact, 0.0, self.air[i])
            self.last_contact[i] = contact
            self.prev[i] = a[i]
            out["reward"][i], out["terms"][i] = tot[0], terms[0]
            out["done"][i], out["trunc"][i] = done, trunc
            if done or trunc:
                out["terminal_obs"][i], out["terminal_mask"][i] = st, True
                self.episode[i] += 1
                self._reset_world(i)
                fr, contact, _ = self._frame(i, np.zeros(12), np.zeros(12), True)
                self.last_contact[i] = contact
                st, pr = self._obs(i, fr, np.zeros(12))
            out["obs"][i], out["priv"][i] = st, pr
        return out
