"""ctypes front-end for the CPU parity oracle (oracle.c).

TEST INFRASTRUCTURE ONLY -- the checker, never the thing measured or shipped.
Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` leg may import this module.  The product package
(paper_2502_08844_b200) never imports it.

Each function restates the reference (deskrl 0.1.0) as cited in oracle.c and
is pinned against tests/golden (generated from the reference itself by
tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

TASK_IDS = {
    "pendulum-swingup": 0,
    "cartpole-balance": 1,
    "acrobot-swingup": 2,
    "reacher-easy": 3,
}
ACTION_DIM = {0: 1, 1: 1, 2: 1, 3: 2}
OBS_DIM = {0: 3, 1: 5, 2: 6, 3: 10}
INFO_DIM = {0: 1, 1: 3, 2: 1, 3: 1}
INFO_KEYS = {0: ("upright",), 1: ("upright", "centered", "still"), 2: ("tip_height",),
             3: ("distance",)}
DEFAULT_DT = {0: 0.01, 1: 0.01, 2: 0.01, 3: 0.005}

# DynamicsParams field order (dynamics.py:40-60)
PARAM_FIELDS = (
    "dt", "gravity", "pend_mass", "pend_length", "pend_damping", "pend_torque_limit",
    "cart_mass", "pole_mass", "pole_length", "rail_limit", "cart_force_limit",
    "link1_mass", "link2_mass", "link1_length", "link2_length", "link_damping",
    "elbow_torque_limit", "reacher_torque_limit",
)
PARAM_DEFAULTS = (0.01, 9.81, 1.0, 0.5, 0.05, 2.5, 1.0, 0.1, 0.5, 1.8, 10.0,
                  1.0, 1.0, 1.0, 1.0, 0.0, 8.0, 1.0)


class _Params(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in PARAM_FIELDS]


class _Cfg(ctypes.Structure):
    _fields_ = [
        ("task", ctypes.c_int32),
        ("wide_init", ctypes.c_int32),
        ("episode_length", ctypes.c_int64),
        ("action_repeat", ctypes.c_int64),
        ("seed", ctypes.c_uint64),
    ]


def build(force: bool = False) -> str:
    srcs = [os.path.join(_HERE, f) for f in ("oracle.c", "locomotion.c", "ppo.c", "Makefile")] + [
        os.path.join(os.path.dirname(_HERE), "paper_2502_08844_b200", "csrc", "ziggurat_tables.h")]
    if force or not os.path.exists(_LIB_PATH) or (
        os.path.getmtime(_LIB_PATH) < max(os.path.getmtime(f) for f in srcs)
    ):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.orc_tol.restype = ctypes.c_double
        _lib.orc_tol.argtypes = [ctypes.c_double] * 4
        _lib.orc_reward.restype = ctypes.c_double
        _lib.orc_batch_step.restype = ctypes.c_int
        _lib.orc_max_threads.restype = ctypes.c_int
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def params_struct(params=None, dt=None) -> _Params:
    vals = list(PARAM_DEFAULTS)
    if params is not None:
        vals = [float(getattr(params, n)) for n in PARAM_FIELDS]
    if dt is not None:
        vals[0] = float(dt)
    return _Params(*vals)


# ---------------------------------------------------------------------------
# primitives


def stream_raw(seed, env_index, episode, step, n) -> np.ndarray:
    out = np.zeros(n, dtype=np.uint64)
    lib().orc_stream_raw(ctypes.c_uint64(seed), ctypes.c_uint64(env_index),
                         ctypes.c_int64(episode), ctypes.c_uint64(step), ctypes.c_int64(n),
                         _p(out))
    return out


def tol(x, lower, upper, margin) -> float:
    return lib().orc_tol(x, lower, upper, margin)


def _cfg(task, episode_length=1000, action_repeat=1, seed=0, wide_init=False) -> _Cfg:
    return _Cfg(TASK_IDS[task] if isinstance(task, str) else task, int(bool(wide_init)),
                episode_length, action_repeat, seed)


def sample_initial(task, seed, env_index, episode, wide_init=False):
    s = np.zeros(4)
    t = np.zeros(2)
    c = _cfg(task, wide_init=wide_init)
    lib().orc_sample_initial(ctypes.byref(c), ctypes.c_uint64(seed), ctypes.c_uint64(env_index),
                             ctypes.c_int64(episode), _p(s), _p(t))
    return s, t


def step_dynamics(task, s, action, params=None, dt=None):
    c = _cfg(task)
    p = params_struct(params, dt if dt is not None else DEFAULT_DT[c.task])
    s = np.ascontiguousarray(s, dtype=np.float64).reshape(4)
    a = np.ascontiguousarray(action, dtype=np.float64).reshape(-1)
    out = np.zeros(4)
    lib().orc_step_dynamics(ctypes.byref(c), ctypes.byref(p), _p(s), _p(a), _p(out))
    return out


def reward(task, s, target=None, params=None):
    c = _cfg(task)
    p = params_struct(params, DEFAULT_DT[c.task])
    s = np.ascontiguousarray(s, dtype=np.float64).reshape(4)
    t = np.zeros(2) if target is None else np.ascontiguousarray(target, dtype=np.float64)
    info = np.zeros(3)
    r = lib().orc_reward(ctypes.byref(c), ctypes.byref(p), _p(s), _p(t), _p(info))
    return r, info[: INFO_DIM[c.task]]


def state_obs(task, s, target=None, params=None):
    c = _cfg(task)
    p = params_struct(params, DEFAULT_DT[c.task])
    s = np.ascontiguousarray(s, dtype=np.float64).reshape(4)
    t = np.zeros(2) if target is None else np.ascontiguousarray(target, dtype=np.float64)
    obs = np.zeros(OBS_DIM[c.task])
    lib().orc_state_obs(ctypes.byref(c), ctypes.byref(p), _p(s), _p(t), _p(obs))
    return obs


# ---------------------------------------------------------------------------
# batched env (BatchEnv semantics, envkit.py:595-650)


class OracleError(Exception):
    def __init__(self, code, index):
        super().__init__(f"oracle step error code {code} at env {index}")
        self.code = code
        self.index = index


@dataclass
class OracleBatchEnv:
    """Mirror of deskrl BatchEnv driven by oracle.c (f64, reference order)."""

    task: str
    num_envs: int
    episode_length: int = 1000
    action_repeat: int = 1
    seed: int = 0
    wide_init: bool = False
    dt: float | None = None
    params: object = None
    env_offset: int = 0

    def __post_init__(self):
        self.tid = TASK_IDS[self.task]
        self.A, self.O, self.I = ACTION_DIM[self.tid], OBS_DIM[self.tid], INFO_DIM[self.tid]
        self._p = params_struct(self.params, self.dt if self.dt is not None
                                else DEFAULT_DT[self.tid])
        n = self.num_envs
        self.state = np.zeros((n, 4))
        self.target = np.zeros((n, 2))
        self.steps = np.zeros(n, dtype=np.int64)
        self.episode = np.full(n, -1, dtype=np.int64)
        self.needs_reset = np.ones(n, dtype=np.uint8)

    def _c(self):
        return _cfg(self.tid, self.episode_length, self.action_repeat, self.seed, self.wide_init)

    def _world(self):
        return (_p(self.state), _p(self.target), _p(self.steps), _p(self.episode),
                _p(self.needs_reset))

    def reset(self, seed=None):
        rewind = 0
        if seed is not None:
            self.seed = int(seed)
            rewind = 1
        obs = np.zeros((self.num_envs, self.O))
        c = self._c()
        lib().orc_batch_reset(ctypes.byref(c), ctypes.byref(self._p),
                              ctypes.c_int64(self.num_envs), ctypes.c_int64(self.env_offset),
                              rewind, *self._world(), _p(obs))
        return obs

    def step(self, actions, autoreset=True):
        a = np.ascontiguousarray(np.asarray(actions, dtype=np.float64).reshape(self.num_envs,
                                                                                self.A))
        n = self.num_envs
        obs = np.zeros((n, self.O))
        rew = np.zeros(n)
        done = np.zeros(n, dtype=np.uint8)
        trunc = np.zeros(n, dtype=np.uint8)
        term = np.zeros((n, self.O))
        mask = np.zeros(n, dtype=np.uint8)
        info = np.zeros((n, self.I))
        err = np.zeros(1, dtype=np.int64)
        c = self._c()
        rc = lib().orc_batch_step(ctypes.byref(c), ctypes.byref(self._p), ctypes.c_int64(n),
                                  ctypes.c_int64(self.env_offset), _p(a), int(bool(autoreset)),
                                  *self._world(), _p(obs), _p(rew), _p(done), _p(trunc),
                                  _p(term), _p(mask), _p(info), _p(err))
        if rc:
            raise OracleError(rc, int(err[0]))
        return obs, rew, done.astype(bool), trunc.astype(bool), term, mask.astype(bool), info

    def rollout(self, actions, nthreads=0):
        """K autoreset steps; actions [K, N, A]; time-major outputs."""
        a = np.ascontiguousarray(actions, dtype=np.float64)
        K = a.shape[0]
        n = self.num_envs
        obs = np.zeros((K, n, self.O))
        rew = np.zeros((K, n))
        done = np.zeros((K, n), dtype=np.uint8)
        trunc = np.zeros((K, n), dtype=np.uint8)
        term = np.zeros((K, n, self.O))
        mask = np.zeros((K, n), dtype=np.uint8)
        info = np.zeros((K, n, self.I))
        c = self._c()
        lib().orc_batch_rollout(ctypes.byref(c), ctypes.byref(self._p), ctypes.c_int64(n),
                                ctypes.c_int64(self.env_offset), ctypes.c_int64(K), _p(a),
                                *self._world(), _p(obs), _p(rew), _p(done), _p(trunc), _p(term),
                                _p(mask), _p(info), int(nthreads))
        return obs, rew, done.astype(bool), trunc.astype(bool), term, mask.astype(bool), info


def max_threads() -> int:
    return int(lib().orc_max_threads())


def use_all_host_threads() -> int:
    """Let the oracle use every core this process may run on (torchrun sets
    OMP_NUM_THREADS=1 for its workers)."""
    n = len(os.sched_getaffinity(0))
    lib().orc_set_threads(n)
    return n
