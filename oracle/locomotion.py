"""ctypes front-end for oracle/locomotion.c (locomotion step tail).

TEST INFRASTRUCTURE ONLY -- the checker (see oracle/oracle.py).
"""

from __future__ import annotations

import ctypes

import numpy as np

from .oracle import lib as _lib

FIELDS = ("base_orientation", "base_lin_vel", "base_ang_vel", "joint_pos", "joint_vel",
          "joint_torque", "foot_height", "foot_height_des", "foot_vel_xy", "foot_contact",
          "airtime", "touchdown", "phase", "command", "action", "prev_action", "joint_nominal",
          "joint_default", "done")
U8 = {"foot_contact", "touchdown", "done"}
# RewardTermConfig field order (rewards.py:51-75)
REWARD_FIELDS = ("w_lin_vel", "sigma_lin_vel", "w_ang_vel", "sigma_ang_vel", "w_airtime",
                 "airtime_min", "airtime_max", "w_clearance", "w_phase", "sigma_phase",
                 "swing_height", "w_slip", "w_orientation", "w_torque", "w_joint_pos",
                 "w_action_rate", "w_energy", "w_pose", "w_termination", "w_standstill",
                 "w_lin_vel_z", "w_ang_vel_xy")
REWARD_DEFAULTS = (1.0, 0.25, 0.5, 0.25, 1.0, 0.1, 0.5, -1.0, 1.0, 0.001, 0.08, -0.1, -1.0,
                   -1e-4, -0.1, -0.01, -1e-3, 0.5, -1.0, -0.1, -0.5, -0.05)


class _Cfg(ctypes.Structure):
    _fields_ = [(f, ctypes.c_double) for f in REWARD_FIELDS] + [("standstill_gated",
                                                                  ctypes.c_int32)]


class _Frames(ctypes.Structure):
    _fields_ = [(f, ctypes.c_void_p) for f in FIELDS] + [("nominal_stride", ctypes.c_int64),
                                                         ("default_stride", ctypes.c_int64)]


def _vp(a):
    return ctypes.c_void_p(a.ctypes.data)


def reward_cfg(**over):
    vals = dict(zip(REWARD_FIELDS, REWARD_DEFAULTS))
    gated = bool(over.pop("standstill_gated", False))
    vals.update(over)
    return _Cfg(*[float(vals[f]) for f in REWARD_FIELDS], int(gated))


def _prep(frames):
    keep = {}
    for f in FIELDS:
        a = np.ascontiguousarray(frames[f], dtype=np.uint8 if f in U8 else np.float64)
        keep[f] = a
    nj = keep["joint_pos"].shape[1]
    n = keep["joint_pos"].shape[0]
    fs = _Frames(*[keep[f].ctypes.data for f in FIELDS],
                 0 if keep["joint_nominal"].ndim == 1 else nj,
                 0 if keep["joint_default"].ndim == 1 else nj)
    return fs, keep, n, nj, keep["foot_height"].shape[1]


def total_reward(frames, **cfg):
    fs, keep, n, nj, nf = _prep(frames)
    c = reward_cfg(**cfg)
    terms = np.zeros((n, 16))
    unc = np.zeros(n)
    tot = np.zeros(n)
    f = _lib().orc_total_reward
    f.restype = ctypes.c_int64
    bad = f(ctypes.c_int64(n), nj, nf, ctypes.byref(c), ctypes.byref(fs),
            terms.ctypes.data_as(ctypes.c_void_p), unc.ctypes.data_as(ctypes.c_void_p),
            tot.ctypes.data_as(ctypes.c_void_p))
    return terms, unc, tot, int(bad)


def loco_obs(frames, prev_action=None, command=None, noise=None, key=(0, 0, 0, 0), pert=None):
    fs, keep, n, nj, nf = _prep(frames)
    pa = np.ascontiguousarray(keep["prev_action"] if prev_action is None else prev_action,
                              dtype=np.float64)
    cm = np.ascontiguousarray(keep["command"] if command is None else command, dtype=np.float64)
    S = 9 + 3 * nj + 3 + 2 * nf
    P = S + nf + nj + 3
    st = np.zeros((n, S))
    pr = np.zeros((n, P))
    nz = None if noise is None else np.ascontiguousarray(noise, dtype=np.float64)
    pt = None if pert is None else np.ascontiguousarray(pert, dtype=np.float64)
    f = _lib().orc_loco_obs
    f.restype = ctypes.c_int64
    seed, env0, ep, step = key
    p = lambda a: None if a is None else a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    bad = f(ctypes.c_int64(n), nj, nf, ctypes.byref(fs), p(pa), p(cm), p(nz),
            ctypes.c_uint64(seed), ctypes.c_int64(env0), ctypes.c_int64(ep),
            ctypes.c_uint64(step), p(pt), p(st), p(pr))
    return st, pr, int(bad)


def project_gravity(q):
    q = np.ascontiguousarray(q, dtype=np.float64)
    n = q.shape[0]
    out = np.zeros((n, 3))
    ok = np.zeros(n, dtype=np.uint8)
    _lib().orc_project_gravity(ctypes.c_int64(n), _vp(q), _vp(out), _vp(ok))
    return out, ok


def pd(params, q_default, a, prev_target, q, v):
    a = np.ascontiguousarray(a, dtype=np.float64)
    n, nj = a.shape
    args = [np.ascontiguousarray(x, dtype=np.float64) for x in (params, q_default, prev_target,
                                                               q, v)]
    tgt = np.zeros((n, nj))
    tau = np.zeros((n, nj))
    _lib().orc_pd(ctypes.c_int64(n), nj, _vp(args[0]), _vp(args[1]), _vp(a),
                  _vp(args[2]), _vp(args[3]), _vp(args[4]), _vp(tgt),
                  _vp(tau))
    return tgt, tau


def progress_clip(raw, hist):
    raw = np.ascontiguousarray(raw, dtype=np.float64)
    hist = np.ascontiguousarray(hist, dtype=np.float64)
    r = np.zeros_like(raw)
    h = np.zeros_like(raw)
    _lib().orc_progress_clip(ctypes.c_int64(raw.size), _vp(raw), _vp(hist),
                             _vp(r), _vp(h))
    return r, h


def wrap_angle(x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.zeros_like(x)
    _lib().orc_wrap_angle(ctypes.c_int64(x.size), _vp(x), _vp(out))
    return out


def advance_phase(phi, freq, dt):
    phi = np.ascontiguousarray(phi, dtype=np.float64)
    n, nf = phi.shape
    fr = np.ascontiguousarray(freq, dtype=np.float64)
    d = np.ascontiguousarray(dt, dtype=np.float64)
    out = np.zeros_like(phi)
    _lib().orc_advance_phase(ctypes.c_int64(n), nf, _vp(phi), _vp(fr),
                             _vp(d), _vp(out))
    return out


def sensor_noise(obs, specs, key):
    """specs: list of (offset, length, scale[, kind]) -- kind "uniform" / "gaussian"."""
    obs = np.ascontiguousarray(obs, dtype=np.float64)
    n, dim = obs.shape
    off = np.array([s[0] for s in specs], dtype=np.int32)
    ln = np.array([s[1] for s in specs], dtype=np.int32)
    sc = np.array([s[2] for s in specs], dtype=np.float64)
    kd = np.array([1 if len(s) > 3 and s[3] == "gaussian" else 0 for s in specs], dtype=np.int32)
    out = np.zeros_like(obs)
    seed, env0, ep, step = key
    _lib().orc_sensor_noise(ctypes.c_int64(n), dim, _vp(obs), len(specs), _vp(off),
                            _vp(ln), _vp(sc), _vp(kd), ctypes.c_uint64(seed),
                            ctypes.c_int64(env0), ctypes.c_int64(ep), ctypes.c_uint64(step),
                            _vp(out))
    return out


def stream_normal(key, count):
    """Generator.standard_normal(count) of stream_rng(*key)."""
    out = np.zeros(count)
    seed, env, ep, step = key
    _lib().orc_stream_normal(ctypes.c_uint64(seed), ctypes.c_uint64(env), ctypes.c_int64(ep),
                             ctypes.c_uint64(step), ctypes.c_int64(count), _vp(out))
    return out


def stream_integers(key, low, high, count):
    """[Generator.integers(low, high) for _ in range(count)] of stream_rng(*key)."""
    out = np.zeros(count, dtype=np.int64)
    seed, env, ep, step = key
    _lib().orc_stream_integers(ctypes.c_uint64(seed), ctypes.c_uint64(env), ctypes.c_int64(ep),
                               ctypes.c_uint64(step), ctypes.c_int64(low), ctypes.c_int64(high),
                               ctypes.c_int64(count), _vp(out))
    return out


DISTRIBUTIONS = {"uniform_additive": 0, "uniform_multiplicative": 1, "log_uniform": 2}


def randomize_params(nominal, ranges, n, key):
    """nominal [F]; ranges: list of (field_index, distribution, low, high).
    Returns (out [n, F], first failing world or -1)."""
    nom = np.ascontiguousarray(nominal, dtype=np.float64)
    fld = np.array([r[0] for r in ranges], dtype=np.int32)
    dst = np.array([DISTRIBUTIONS[r[1]] for r in ranges], dtype=np.int32)
    lo = np.array([r[2] for r in ranges], dtype=np.float64)
    hi = np.array([r[3] for r in ranges], dtype=np.float64)
    out = np.zeros((n, nom.size))
    seed, env0, ep, step = key
    lib = _lib()
    lib.orc_randomize_params.restype = ctypes.c_int64
    fail = lib.orc_randomize_params(ctypes.c_int64(n), nom.size, _vp(nom), len(ranges), _vp(fld),
                                    _vp(dst), _vp(lo), _vp(hi), ctypes.c_uint64(seed),
                                    ctypes.c_int64(env0), ctypes.c_int64(ep),
                                    ctypes.c_uint64(step), _vp(out))
    return out, int(fail)


class DelayLines:
    """n batched DelayLine rings (randomization.py:27-62) for oracle checks."""

    def __init__(self, n, dim, min_delay, max_delay, per_step=False):
        self.n, self.dim, self.lo, self.hi, self.per_step = n, dim, min_delay, max_delay, per_step
        self.ring = np.zeros((n, max_delay + 1, dim))
        self.head = np.zeros(n, np.int32)
        self.count = np.zeros(n, np.int32)
        self.delay = np.zeros(n, np.int32)

    def reset(self, key):
        seed, env0, ep, step = key
        _lib().orc_delay_reset(ctypes.c_int64(self.n), self.lo, self.hi, ctypes.c_uint64(seed),
                               ctypes.c_int64(env0), ctypes.c_int64(ep), ctypes.c_uint64(step),
                               _vp(self.delay), _vp(self.count), _vp(self.head))

    def push_pop(self, value, key):
        v = np.ascontiguousarray(value, dtype=np.float64).reshape(self.n, self.dim)
        out = np.zeros_like(v)
        seed, env0, ep, step = key
        _lib().orc_delay_push_pop(ctypes.c_int64(self.n), self.dim, self.lo, self.hi,
                                  int(self.per_step), _vp(self.ring), _vp(self.head),
                                  _vp(self.count), _vp(self.delay), ctypes.c_uint64(seed),
                                  ctypes.c_int64(env0), ctypes.c_int64(ep), ctypes.c_uint64(step),
                                  _vp(v), _vp(out))
        return out


def pose_injection(pose, bounds, prob, key):
    pose = np.ascontiguousarray(pose, dtype=np.float64)
    n, dim = pose.shape
    b = np.ascontiguousarray(bounds, dtype=np.float64)
    out = np.zeros_like(pose)
    seed, env0, ep, step = key
    _lib().orc_pose_injection(ctypes.c_int64(n), dim, _vp(pose), _vp(b),
                              ctypes.c_double(prob), ctypes.c_uint64(seed), ctypes.c_int64(env0),
                              ctypes.c_int64(ep), ctypes.c_uint64(step), _vp(out))
    return out


def curriculum(state, success, max_level, threshold):
    st = np.ascontiguousarray(state, dtype=np.int64).copy()
    s = np.ascontiguousarray(success, dtype=np.uint8)
    _lib().orc_curriculum(ctypes.c_int64(st.shape[0]), _vp(st), _vp(s),
                          ctypes.c_int64(max_level), ctypes.c_int64(threshold))
    return st
