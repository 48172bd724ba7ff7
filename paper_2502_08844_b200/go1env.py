"""Go1 joystick environment on B200: articulated physics with the locomotion
step tail fused into the same kernel (csrc/go1env.cuh; C ABI dk_go1_*).

``DeviceGo1Env`` presents the batched-env surface of the reference's BatchEnv
(envkit.py:595-650) for the Go1 joystick task the reference itself leaves out
of scope: ``reset(seed)`` -> observation dict, ``step(actions)`` ->
(obs, reward, done, trunc, info) with auto-reset and the terminal observation,
plus ``rollout(actions[K])`` fusing K control steps into one launch.
Observations use build_locomotion_observation's Go1 layout: ``state`` [N, 56]
(noisy) and ``privileged_state`` [N, 75] (clean + contacts, torques,
perturbation).  Parity: physics vs oracle/physics.c, tail vs
oracle/locomotion.c, the composition vs oracle/go1env.py -- UNPINNED.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

from . import _native as nat
from .envkit import ConfigError, _check
from .locomotion import RewardTermConfig, _reward_cfg
from .physmodel import PhysModel, go1_model

OBS_DIM, PRIV_DIM, ACTION_DIM, NUM_TERMS = 56, 75, 12, 16


class Go1ConfigC(ctypes.Structure):
    _fields_ = [("episode_length", ctypes.c_int64), ("ctrl_dt", ctypes.c_double),
                ("action_scale", ctypes.c_double), ("gait_freq", ctypes.c_double),
                ("term_height", ctypes.c_double), ("cmd_lo", ctypes.c_double * 3),
                ("cmd_hi", ctypes.c_double * 3), ("joint_noise", ctypes.c_double),
                ("yaw_range", ctypes.c_double), ("obs_noise", ctypes.c_double * 5),
                ("seed", ctypes.c_uint64), ("reward", nat.RewardConfigC),
                ("dr_friction", ctypes.c_double * 2), ("dr_payload", ctypes.c_double * 2),
                ("dr_kp_scale", ctypes.c_double * 2)]


@dataclass
class Go1Config:
    """dk_go1_config (include/deskrl_b200.h); defaults = dk_go1_default_config."""

    episode_length: int = 1000
    ctrl_dt: float = 0.02
    action_scale: float = 0.5
    gait_freq: float = 1.5
    term_height: float = 0.12
    cmd_lo: tuple = (-1.5, -0.8, -1.2)
    cmd_hi: tuple = (1.5, 0.8, 1.2)
    joint_noise: float = 0.1
    yaw_range: float = math.pi
    obs_noise: tuple = (0.05, 0.1, 0.2, 0.01, 1.5)  # ObservationNoise (envkit.py:138-144)
    seed: int = 0
    reward: RewardTermConfig = field(default_factory=RewardTermConfig)
    # per-world domain randomisation at every reset (friction, payload kg, kp scale)
    dr_friction: tuple = (0.4, 1.0)
    dr_payload: tuple = (-0.5, 1.5)
    dr_kp_scale: tuple = (0.9, 1.1)

    def to_c(self) -> Go1ConfigC:
        c = Go1ConfigC()
        c.episode_length = int(self.episode_length)
        for f in ("ctrl_dt", "action_scale", "gait_freq", "term_height", "joint_noise",
                  "yaw_range"):
            setattr(c, f, float(getattr(self, f)))
        for k in range(3):
            c.cmd_lo[k], c.cmd_hi[k] = float(self.cmd_lo[k]), float(self.cmd_hi[k])
        for k in range(5):
            c.obs_noise[k] = float(self.obs_noise[k])
        c.seed = int(self.seed) & (2**64 - 1)
        c.reward = _reward_cfg(self.reward)
        for k in range(2):
            c.dr_friction[k] = float(self.dr_friction[k])
            c.dr_payload[k] = float(self.dr_payload[k])
            c.dr_kp_scale[k] = float(self.dr_kp_scale[k])
        return c

    def oracle_dict(self) -> dict:
        """the same configuration for oracle/go1env.py (test infrastructure)"""
        rw = {f: getattr(self.reward, f) for f in nat.REWARD_FIELDS}
        rw["standstill_gated"] = bool(self.reward.standstill_gated)
        return dict(episode_length=self.episode_length, ctrl_dt=self.ctrl_dt,
                    action_scale=self.action_scale, gait_freq=self.gait_freq,
                    term_height=self.term_height, cmd_lo=tuple(self.cmd_lo),
                    cmd_hi=tuple(self.cmd_hi), joint_noise=self.joint_noise,
                    yaw_range=self.yaw_range, obs_noise=tuple(self.obs_noise), seed=self.seed,
                    reward=rw, dr_friction=tuple(self.dr_friction),
                    dr_payload=tuple(self.dr_payload), dr_kp_scale=tuple(self.dr_kp_scale))


class DeviceGo1Env:
    """N Go1 joystick worlds on one GPU; CUDA tensors in and out, enqueued on
    the current stream (``check()`` synchronises and raises pending errors)."""

    def __init__(self, num_envs: int, config: Go1Config | None = None,
                 model: PhysModel | None = None, dtype="float32", device: int | None = None,
                 env_index_offset: int = 0):
        import torch

        self._torch = torch
        self.num_envs = int(num_envs)
        if self.num_envs < 1:
            raise ConfigError("num_envs must be >= 1")
        self.config = config or Go1Config()
        self.model = (model or go1_model()).validate()
        self.action_dim, self.obs_dim, self.priv_dim = ACTION_DIM, OBS_DIM, PRIV_DIM
        self.env_index_offset = int(env_index_offset)
        if dtype in ("float32", torch.float32):
            self.dtype, code = torch.float32, nat.DK_F32
        elif dtype in ("float64", torch.float64):
            self.dtype, code = torch.float64, nat.DK_F64
        else:
            raise ConfigError(f"unsupported dtype {dtype!r}")
        if device is None:
            device = torch.cuda.current_device() if torch.cuda.is_available() else 0
        self.device = torch.device("cuda", int(device))
        self._lib = nat.lib()
        self._mc, self._cc = self.model.to_c(), self.config.to_c()
        h = ctypes.c_void_p()
        _check(self._lib.dk_go1_create(ctypes.byref(self._mc), ctypes.byref(self._cc), code,
                                       self.num_envs, self.env_index_offset, int(device),
                                       ctypes.byref(h)))
        self.h = h

    def _stream(self):
        return ctypes.c_void_p(self._torch.cuda.current_stream(self.device).cuda_stream)

    @staticmethod
    def _p(t):
        return None if t is None else t.data_ptr()

    def outputs(self, K: int | None, with_priv=True, with_terms=False, with_terminal=True,
                with_terminal_priv=False):
        torch = self._torch
        lead = () if K is None else (int(K),)
        n, dt, dev = self.num_envs, self.dtype, self.device
        e = lambda *s, d=dt: torch.empty(lead + (n,) + s, dtype=d, device=dev)  # noqa: E731
        u8 = torch.uint8
        return {"obs": e(OBS_DIM), "privileged_state": e(PRIV_DIM) if with_priv else None,
                "reward": e(), "done": e(d=u8), "trunc": e(d=u8),
                "terms": e(NUM_TERMS) if with_terms else None,
                "terminal_obs": e(OBS_DIM) if with_terminal else None,
                "terminal_privileged_state": e(PRIV_DIM) if with_terminal_priv else None,
                "terminal_mask": e(d=u8) if with_terminal else None}

    def _outputs(self, lead, with_info):
        """DeviceBatchEnv-style reusable step buffers (collect_rollout_device): one
        step, with the terminal privileged rows an asymmetric critic bootstraps from."""
        return self.outputs(None, with_terminal_priv=True)

    def reset(self, seed: int | None = None) -> dict:
        torch = self._torch
        if seed is not None:
            self.config.seed = int(seed)
        obs = torch.empty((self.num_envs, OBS_DIM), dtype=self.dtype, device=self.device)
        priv = torch.empty((self.num_envs, PRIV_DIM), dtype=self.dtype, device=self.device)
        _check(self._lib.dk_go1_reset(self.h, int(seed is not None),
                                      0 if seed is None else int(seed) & (2**64 - 1),
                                      obs.data_ptr(), priv.data_ptr(), self._stream()))
        return {"state": obs, "privileged_state": priv}

    def rollout(self, actions, out: dict | None = None, with_terms=False) -> dict:
        """K control steps in one launch; actions [K, N, 12]."""
        torch = self._torch
        a = torch.as_tensor(actions, device=self.device, dtype=self.dtype)
        if a.dim() != 3 or tuple(a.shape[1:]) != (self.num_envs, ACTION_DIM):
            raise ConfigError(f"actions must be [K, {self.num_envs}, {ACTION_DIM}]")
        a = a.contiguous()
        K = int(a.shape[0])
        o = out or self.outputs(K, with_terms=with_terms)
        _check(self._lib.dk_go1_step_ex(
            self.h, K, a.data_ptr(), o["obs"].data_ptr(), self._p(o.get("privileged_state")),
            o["reward"].data_ptr(), o["done"].data_ptr(), o["trunc"].data_ptr(),
            self._p(o.get("terms")), self._p(o.get("terminal_obs")),
            self._p(o.get("terminal_privileged_state")), self._p(o.get("terminal_mask")),
            self._stream()))
        self._keep = a
        return o

    def step(self, actions, out: dict | None = None, with_terms=False, autoreset=True,
             with_info=False) -> dict:
        """One control step; actions [N, 12]; outputs without the K axis.  (The
        episode auto-resets always; ``autoreset`` / ``with_info`` are accepted
        for collect_rollout_device's DeviceBatchEnv-style calls.)"""
        if not autoreset:
            raise ConfigError("DeviceGo1Env always auto-resets")
        a = self._torch.as_tensor(actions, device=self.device, dtype=self.dtype)
        o = out or self.outputs(None, with_terms=with_terms)
        view = {k: (v.unsqueeze(0) if v is not None else None) for k, v in o.items()}
        self.rollout(a.unsqueeze(0), out=view)
        return o

    def state(self) -> dict:
        torch = self._torch
        n, dt, dev = self.num_envs, self.dtype, self.device
        s = {"qpos": torch.empty((n, 19), dtype=dt, device=dev),
             "qvel": torch.empty((n, 18), dtype=dt, device=dev),
             "command": torch.empty((n, 3), dtype=dt, device=dev),
             "phase": torch.empty((n, 4), dtype=dt, device=dev),
             "airtime": torch.empty((n, 4), dtype=dt, device=dev),
             "last_contact": torch.empty((n, 4), dtype=torch.uint8, device=dev),
             "prev_action": torch.empty((n, 12), dtype=dt, device=dev),
             "steps": torch.empty((n,), dtype=torch.int32, device=dev),
             "episode": torch.empty((n,), dtype=torch.int32, device=dev)}
        _check(self._lib.dk_go1_get_state(self.h, *[s[k].data_ptr() for k in (
            "qpos", "qvel", "command", "phase", "airtime", "last_contact", "prev_action",
            "steps", "episode")], self._stream()))
        return s

    def params(self):
        """[N, 3]: each world's friction, trunk mass and kp this episode"""
        p = self._torch.empty((self.num_envs, 3), dtype=self.dtype, device=self.device)
        _check(self._lib.dk_go1_get_params(self.h, p.data_ptr(), self._stream()))
        return p

    def check(self):
        self._torch.cuda.current_stream(self.device).synchronize()
        k, i = ctypes.c_int64(-1), ctypes.c_int64(-1)
        rc = self._lib.dk_go1_check(self.h, ctypes.byref(k), ctypes.byref(i))
        if rc != nat.DK_OK:
            from .envkit import _ERR, BackendError

            err = _ERR.get(rc, BackendError)(nat.last_error())
            err.step_index, err.env_index = int(k.value), int(i.value)
            raise err

    @property
    def kernel_launches(self) -> int:
        return int(self._lib.dk_go1_kernel_launches(self.h))

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self._lib.dk_go1_destroy(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


__all__ = ["ACTION_DIM", "DeviceGo1Env", "Go1Config", "NUM_TERMS", "OBS_DIM", "PRIV_DIM"]
