"""Locomotion step tail on B200, batched.

Mirrors the reference's per-frame pure functions over batches of frames held
as CUDA tensors, computed by the sm_100a kernels of libdeskrl_b200.so:

* ``locomotion_tail`` -- ``rewards.total_reward`` (rewards.py:201-211, 16 terms
  97-177) fused with ``envkit.build_locomotion_observation`` (envkit.py:147-193)
  in one pass over the frames; ``total_reward_batch`` and
  ``build_locomotion_observation_batch`` are the two halves with the
  reference's return shapes.
* ``pd_batch`` -- ``action_to_target`` + ``pd_torque`` (envkit.py:111-131).
* ``advance_phase_batch`` -- ``advance_phase`` + ``phase_encode``
  (mathcore.py:143-177).
* ``progress_clip_reward_batch`` (envkit.py:196-202).
* ``apply_sensor_noise_batch`` (uniform and gaussian), ``randomize_params_batch``,
  ``DelayLineBatch``, ``pose_injection_batch``, ``curriculum_update_batch``
  (randomization.py:27-62, 88-108, 156-181, 188-199, 224-238).

Randomness: the reference takes caller-supplied numpy Generators; here each
world's stream is ``stream_rng(seed, env_index_offset + world, episode, step)``
(envkit.py:41-49, the reference's own keying), bit-compatible with NumPy.

A batch of frames is a dict of tensors named like ``LocomotionFrame`` fields
(rewards.py:17-44), each ``[R, dim]`` (``foot_vel_xy`` ``[R, F, 2]``; flags
bool/uint8; ``joint_nominal`` / ``joint_default`` may be one ``[J]`` row).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .envkit import ConfigError, InvalidInputError, _check

TERM_NAMES = ("lin_vel_tracking", "ang_vel_tracking", "feet_airtime", "feet_clearance",
              "feet_phase", "feet_slip", "orientation", "joint_torque", "joint_position",
              "action_rate", "energy", "pose", "termination", "standstill", "lin_vel_z",
              "ang_vel_xy")  # TERM_REGISTRY order (rewards.py:181-198)
_WEIGHT_OF = dict(zip(TERM_NAMES, ("w_lin_vel", "w_ang_vel", "w_airtime", "w_clearance",
                                   "w_phase", "w_slip", "w_orientation", "w_torque",
                                   "w_joint_pos", "w_action_rate", "w_energy", "w_pose",
                                   "w_termination", "w_standstill", "w_lin_vel_z",
                                   "w_ang_vel_xy")))


@dataclass(frozen=True)
class RewardTermConfig:
    """Weights, kernel scales and gait constants (reference: rewards.py:47-81)."""

    w_lin_vel: float = 1.0
    sigma_lin_vel: float = 0.25
    w_ang_vel: float = 0.5
    sigma_ang_vel: float = 0.25
    w_airtime: float = 1.0
    airtime_min: float = 0.1
    airtime_max: float = 0.5
    w_clearance: float = -1.0
    w_phase: float = 1.0
    sigma_phase: float = 0.001
    swing_height: float = 0.08
    w_slip: float = -0.1
    w_orientation: float = -1.0
    w_torque: float = -1e-4
    w_joint_pos: float = -0.1
    w_action_rate: float = -0.01
    w_energy: float = -1e-3
    w_pose: float = 0.5
    w_termination: float = -1.0
    w_standstill: float = -0.1
    w_lin_vel_z: float = -0.5
    w_ang_vel_xy: float = -0.05
    standstill_gated: bool = False

    def __post_init__(self):
        if self.sigma_lin_vel <= 0 or self.sigma_ang_vel <= 0 or self.sigma_phase <= 0:
            raise ValueError("kernel scales must be positive")
        if self.airtime_min > self.airtime_max:
            raise ValueError("airtime_min must not exceed airtime_max")


@dataclass(frozen=True)
class ObservationNoise:
    """Uniform noise scales per signal group (reference: envkit.py:138-144)."""

    gravity: float = 0.0
    lin_vel: float = 0.0
    ang_vel: float = 0.0
    joint_pos: float = 0.0
    joint_vel: float = 0.0


@dataclass(frozen=True)
class PDParams:
    """PD action mapping (reference: envkit.py:91-108)."""

    kp: float
    kd: float
    action_scale: float
    q_default: object
    mode: str = "absolute"
    torque_limit: float = float("inf")
    joint_range: tuple = (-float("inf"), float("inf"))

    def __post_init__(self):
        if self.kp < 0 or self.kd < 0:
            raise InvalidInputError("PD gains must be non-negative")
        if self.action_scale <= 0:
            raise InvalidInputError("action scale must be positive")
        if self.mode not in ("absolute", "relative"):
            raise InvalidInputError(f"unknown PD mode {self.mode!r}")


@dataclass(frozen=True)
class NoiseKey:
    """Philox stream key: stream_rng(seed, env_index_offset + world, episode, step)."""

    seed: int = 0
    env_index_offset: int = 0
    episode: object = None  # None (episode 0) or a CUDA uint32/int tensor [num_worlds]
    step: int = 0


# ---------------------------------------------------------------------------
# helpers


def _torch():
    import torch

    return torch


def _dtype_code(t):
    torch = _torch()
    if t.dtype == torch.float64:
        return nat.DK_F64
    if t.dtype == torch.float32:
        return nat.DK_F32
    raise ConfigError(f"unsupported dtype {t.dtype} (float32 or float64)")


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(dev):
    return ctypes.c_void_p(_torch().cuda.current_stream(dev).cuda_stream)


_CONST_CACHE: dict = {}


def _const(key, make):
    """Small per-call constant tensors (joint defaults, noise-spec tables) cached on
    the device by value, so repeated calls issue no host-to-device copies."""
    t = _CONST_CACHE.get(key)
    if t is None:
        if len(_CONST_CACHE) > 256:
            _CONST_CACHE.clear()
        t = _CONST_CACHE[key] = make()
    return t


def _key(key: NoiseKey, n_worlds, dev):
    torch = _torch()
    ep = None
    if key.episode is not None:
        ep = torch.as_tensor(key.episode, device=dev).to(torch.int64).remainder(2**32)
        ep = ep.to(torch.int32).contiguous()  # same bits as uint32
        if ep.numel() != n_worlds:
            raise InvalidInputError("episode must have one entry per world")
    c = nat.NoiseKeyC(int(key.seed) & (2**64 - 1), int(key.env_index_offset),
                      None if ep is None else ep.data_ptr(), int(key.step) & (2**64 - 1))
    return c, ep


def _reward_cfg(cfg: RewardTermConfig):
    return nat.RewardConfigC(*[float(getattr(cfg, f)) for f in nat.REWARD_FIELDS],
                             int(bool(cfg.standstill_gated)), 0)


def _prep_frames(frames, dtype, dev):
    torch = _torch()
    keep = {}
    for f in nat.FRAME_FIELDS:
        if f not in frames:
            raise InvalidInputError(f"frame batch is missing field {f!r}")
        t = torch.as_tensor(frames[f], device=dev)
        if f in ("foot_contact", "touchdown", "done"):
            t = t.to(torch.uint8)
        else:
            t = t.to(dtype)
        keep[f] = t.contiguous()
    R, J = keep["joint_pos"].shape
    F = keep["foot_height"].shape[1]
    shapes = {"base_orientation": (R, 4), "base_lin_vel": (R, 3), "base_ang_vel": (R, 3),
              "joint_vel": (R, J), "joint_torque": (R, J), "foot_height_des": (R, F),
              "foot_vel_xy": (R, F, 2), "foot_contact": (R, F), "airtime": (R, F),
              "touchdown": (R, F), "phase": (R, F), "command": (R, 3), "action": (R, J),
              "prev_action": (R, J), "done": (R,)}
    for f, shp in shapes.items():
        if tuple(keep[f].shape) != shp:
            raise InvalidInputError(f"{f} must have shape {shp}, got {tuple(keep[f].shape)}")
    strides = []
    for f in ("joint_nominal", "joint_default"):
        shp = tuple(keep[f].shape)
        if shp == (J,):
            strides.append(0)
        elif shp == (R, J):
            strides.append(J)
        else:
            raise InvalidInputError(f"{f} must have shape {(J,)} or {(R, J)}")
    c = nat.LocoFramesC(*[keep[f].data_ptr() for f in nat.FRAME_FIELDS], *strides)
    return c, keep, R, J, F


def frames_from_reference(frames, device="cuda", dtype="float64"):
    """Stack a list of LocomotionFrame-like objects into a device batch."""
    torch = _torch()
    tdt = torch.float64 if str(dtype).endswith("64") else torch.float32
    out = {}
    for f in nat.FRAME_FIELDS:
        vals = [getattr(fr, f) for fr in frames]
        if f in ("foot_contact", "touchdown", "done"):
            arr = np.array([np.asarray(v, dtype=bool) for v in vals], dtype=np.uint8)
            out[f] = torch.as_tensor(arr, device=device)
        else:
            out[f] = torch.as_tensor(np.array(vals, dtype=np.float64), device=device, dtype=tdt)
    return out


# ---------------------------------------------------------------------------
# B1 + B2 (+ B3, B4 inside): the fused tail


def locomotion_tail(frames, cfg: RewardTermConfig | None = None, prev_action=None, command=None,
                    noise: ObservationNoise | None = None, key: NoiseKey | None = None,
                    perturbation=None, num_worlds: int | None = None, with_terms=True,
                    with_obs=True, check=True):
    """Reward breakdown and observation slots of R = K * num_worlds frames.

    Rows are step-major ([K][num_worlds]); row block k draws its noise at
    step ``key.step + k``.  Returns a dict of CUDA tensors: ``total``,
    ``unclipped``, ``terms`` [R,16] (TERM_REGISTRY order), ``state``
    [R, 9+3J+3+2F] (noisy policy view) and ``privileged_state``.
    """
    torch = _torch()
    cfg = cfg or RewardTermConfig()
    key = key or NoiseKey()
    dtype = torch.as_tensor(frames["joint_pos"]).dtype
    if dtype not in (torch.float32, torch.float64):
        dtype = torch.float64
    dev = torch.as_tensor(frames["joint_pos"]).device
    if dev.type != "cuda":
        raise InvalidInputError("frames must be CUDA tensors")
    fc, keep, R, J, F = _prep_frames(frames, dtype, dev)
    N = R if num_worlds is None else int(num_worlds)
    if N <= 0 or R % N:
        raise InvalidInputError("rows must be a multiple of num_worlds")
    K = R // N

    def opt(t, shape):
        if t is None:
            return None
        t = torch.as_tensor(t, device=dev).to(dtype).contiguous()
        if tuple(t.shape) != shape:
            raise InvalidInputError(f"expected shape {shape}, got {tuple(t.shape)}")
        return t

    pa, cm, pt = opt(prev_action, (R, J)), opt(command, (R, 3)), opt(perturbation, (R, 3))
    S = 9 + 3 * J + 3 + 2 * F
    P = S + F + J + 3
    out = {"total": torch.empty(R, device=dev, dtype=dtype),
           "unclipped": torch.empty(R, device=dev, dtype=dtype),
           "terms": torch.empty((R, 16), device=dev, dtype=dtype) if with_terms else None,
           "state": torch.empty((R, S), device=dev, dtype=dtype) if with_obs else None,
           "privileged_state": torch.empty((R, P), device=dev, dtype=dtype) if with_obs else None}
    oc = nat.LocoOutputsC(*[None if out[k] is None else out[k].data_ptr()
                            for k in ("total", "unclipped", "terms", "state",
                                      "privileged_state")])
    nz = None
    if noise is not None:
        nz = (ctypes.c_double * 5)(noise.gravity, noise.lin_vel, noise.ang_vel, noise.joint_pos,
                                   noise.joint_vel)
    kc, ep = _key(key, N, dev)
    bad = torch.full((1,), -1, dtype=torch.int64, device=dev)
    rc = nat.lib().dk_loco_tail(_dtype_code(keep["joint_pos"]), K, N, J, F,
                                ctypes.byref(_reward_cfg(cfg)), ctypes.byref(fc), _ptr(pa),
                                _ptr(cm), nz, ctypes.byref(kc), _ptr(pt), ctypes.byref(oc),
                                _ptr(bad), _stream(dev))
    _check(rc)
    # (inputs may be freed on return: torch's caching allocator only reuses
    # their blocks for work ordered after this launch on the same stream)
    if check and int(bad.item()) != -1:
        raise InvalidInputError("quaternion is not unit length")
    return out


@dataclass
class RewardBreakdownBatch:
    """rewards.RewardBreakdown (rewards.py:84-89) for a batch."""

    terms: dict
    weighted: dict
    unclipped_total: object
    total: object


def total_reward_batch(frames, cfg: RewardTermConfig | None = None, **kw) -> RewardBreakdownBatch:
    cfg = cfg or RewardTermConfig()
    o = locomotion_tail(frames, cfg, with_obs=False, **kw)
    terms = {name: o["terms"][:, k] for k, name in enumerate(TERM_NAMES)}
    weighted = {name: getattr(cfg, _WEIGHT_OF[name]) * terms[name] for name in TERM_NAMES}
    return RewardBreakdownBatch(terms, weighted, o["unclipped"], o["total"])


def build_locomotion_observation_batch(frames, prev_action, command, noise=None, key=None,
                                       perturbation_force=None, **kw) -> dict:
    o = locomotion_tail(frames, RewardTermConfig(), prev_action=prev_action, command=command,
                        noise=noise, key=key, perturbation=perturbation_force, with_terms=False,
                        **kw)
    return {"state": o["state"], "privileged_state": o["privileged_state"]}


# ---------------------------------------------------------------------------
# B5 / B4 / B6


def pd_batch(action, prev_target, q, qd, p: PDParams):
    """(target, torque) = action_to_target + pd_torque for [n, J] tensors."""
    torch = _torch()
    a = action.contiguous()
    dt = a.dtype
    n, J = a.shape
    dev = a.device
    qd64 = tuple(float(v) for v in np.asarray(p.q_default, dtype=np.float64).reshape(-1))
    qdef = _const(("qdef", qd64, str(dev), str(dt)),
                  lambda: torch.tensor(qd64, dtype=torch.float64, device=dev).to(dt))
    if qdef.shape != (J,):
        raise InvalidInputError("q_default must have one entry per joint")
    q = q.to(dt).contiguous()
    qd = qd.to(dt).contiguous()
    if q.shape != a.shape or qd.shape != a.shape:
        raise InvalidInputError("pd_torque: mismatched dimensions")
    prev = None if prev_target is None else prev_target.to(dt).contiguous()
    params = (ctypes.c_double * 7)(p.kp, p.kd, p.action_scale, p.torque_limit, p.joint_range[0],
                                   p.joint_range[1], 1.0 if p.mode == "relative" else 0.0)
    target = torch.empty_like(a)
    torque = torch.empty_like(a)
    _check(nat.lib().dk_loco_pd(_dtype_code(a), n, J, params, _ptr(qdef), _ptr(a), _ptr(prev),
                                _ptr(q), _ptr(qd), _ptr(target), _ptr(torque), _stream(dev)))
    return target, torque


def advance_phase_batch(phi, frequency, dt):
    """(wrapped phase, (cos, sin) pairs) for phi [n, F]; frequency / dt scalar or [n]."""
    torch = _torch()
    phi = phi.contiguous()
    n, F = phi.shape
    def per_world(v, tag):
        if isinstance(v, (int, float)):
            return _const((tag, float(v), n, str(phi.device), str(phi.dtype)),
                          lambda: torch.full((n,), float(v), device=phi.device, dtype=phi.dtype))
        return torch.as_tensor(v, device=phi.device, dtype=phi.dtype).expand(n).contiguous()

    fr = per_world(frequency, "freq")
    d = per_world(dt, "dt")
    out = torch.empty_like(phi)
    cs = torch.empty((n, F, 2), device=phi.device, dtype=phi.dtype)
    _check(nat.lib().dk_loco_phase(_dtype_code(phi), n, F, _ptr(phi), _ptr(fr), _ptr(d),
                                   _ptr(out), _ptr(cs), _stream(phi.device)))
    return out, cs


def progress_clip_reward_batch(raw, history_max):
    """(reward, new history_max) elementwise (envkit.py:196-202)."""
    raw = raw.contiguous()
    hist = history_max.to(raw.dtype).clone()
    rew = raw.new_empty(raw.shape)
    _check(nat.lib().dk_loco_progress_clip(_dtype_code(raw), raw.numel(), _ptr(raw), _ptr(hist),
                                           _ptr(rew), _stream(raw.device)))
    return rew, hist


# ---------------------------------------------------------------------------
# B7: domain randomisation primitives


_NOISE_KINDS = {"uniform": 0, "gaussian": 1}


def apply_sensor_noise_batch(obs: dict, specs, key: NoiseKey):
    """randomization.apply_sensor_noise for batched slots, both kinds.

    ``obs``: slot name -> CUDA tensor [n, d]; ``specs``: objects with
    ``slot``, ``scale``, ``kind`` (NoiseSpec, randomization.py:73-85): uniform
    U(-scale, scale) or gaussian Generator.normal(0, scale), drawn in spec order
    from each world's stream (bit-compatible with NumPy).
    """
    torch = _torch()
    names = list(obs)
    for spec in specs:
        if spec.slot.startswith("privileged"):
            raise ConfigError("privileged slots must stay noise-free")
        if spec.slot not in obs:
            raise ConfigError(f"unknown observation slot {spec.slot!r}")
        kind = getattr(spec, "kind", "uniform")
        if kind not in _NOISE_KINDS:
            raise ConfigError(f"unknown noise kind {kind!r}")
        if spec.scale < 0:
            raise ConfigError("noise scale must be non-negative")
    first = obs[names[0]]
    n = first.shape[0]
    dt = first.dtype
    flat, offs = [], {}
    o = 0
    for k in names:
        t = obs[k].to(dt).reshape(n, -1)
        offs[k] = (o, t.shape[1])
        o += t.shape[1]
        flat.append(t)
    buf = torch.cat(flat, 1).contiguous()
    dev = first.device
    table = tuple((offs[s.slot][0], offs[s.slot][1], float(s.scale),
                   _NOISE_KINDS[getattr(s, "kind", "uniform")]) for s in specs)

    def make_tables():
        return (torch.tensor([t[0] for t in table], dtype=torch.int32, device=dev),
                torch.tensor([t[1] for t in table], dtype=torch.int32, device=dev),
                torch.tensor([t[2] for t in table], dtype=torch.float64, device=dev),
                torch.tensor([t[3] for t in table], dtype=torch.int32, device=dev))

    off, ln, sc, kd = _const(("noise", table, str(dev)), make_tables)
    kc, ep = _key(key, n, dev)
    _check(nat.lib().dk_dr_sensor_noise(_dtype_code(buf), n, buf.shape[1], _ptr(buf), len(specs),
                                        _ptr(off), _ptr(ln), _ptr(sc), _ptr(kd),
                                        ctypes.byref(kc), _stream(dev)))
    out = dict(obs)
    for k in names:
        a, b = offs[k]
        if any(s.slot == k for s in specs):
            out[k] = buf[:, a:a + b].reshape(obs[k].shape)
    return out


_DISTRIBUTIONS = {"uniform_additive": 0, "uniform_multiplicative": 1, "log_uniform": 2}


def randomize_params_batch(nominal, spec, key: NoiseKey, num_worlds: int, device=None):
    """randomization.randomize_params for ``num_worlds`` worlds at once.

    ``nominal``: a dataclass of floats (e.g. DynamicsParams); ``spec``: an
    object with ``params`` = ParamRange-like (path, distribution, low, high).
    World w draws from stream_rng(seed, env_index_offset + w, episode, step),
    so row w equals ``randomize_params(nominal, spec, stream_rng(...))``.
    Returns (params [num_worlds, F] float64 CUDA tensor, field names).
    """
    import dataclasses

    torch = _torch()
    names = [f.name for f in dataclasses.fields(nominal)]
    ranges = list(getattr(spec, "params", ()))
    for pr in ranges:
        if pr.path not in names:
            raise ConfigError(f"unknown parameter path {pr.path!r}")
        if pr.distribution not in _DISTRIBUTIONS:
            raise ConfigError(f"unknown distribution {pr.distribution!r}")
        if pr.low > pr.high:
            raise ConfigError(f"bounds out of order for {pr.path!r}")
        if pr.distribution != "uniform_additive" and pr.low <= 0:
            raise ConfigError("multiplicative/log bounds must be positive")
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    nom = torch.tensor([float(getattr(nominal, k)) for k in names], dtype=torch.float64,
                       device=dev)
    out = torch.empty((num_worlds, len(names)), dtype=torch.float64, device=dev)
    if not ranges:
        out.copy_(nom.expand(num_worlds, -1))
        return out, names
    lo = [float(np.log(pr.low)) if pr.distribution == "log_uniform" else float(pr.low)
          for pr in ranges]  # np.log as the reference computes it (randomization.py:175)
    hi = [float(np.log(pr.high)) if pr.distribution == "log_uniform" else float(pr.high)
          for pr in ranges]
    fld = torch.tensor([names.index(pr.path) for pr in ranges], dtype=torch.int32, device=dev)
    dst = torch.tensor([_DISTRIBUTIONS[pr.distribution] for pr in ranges], dtype=torch.int32,
                       device=dev)
    lo_t = torch.tensor(lo, dtype=torch.float64, device=dev)
    hi_t = torch.tensor(hi, dtype=torch.float64, device=dev)
    fail = torch.full((1,), -1, dtype=torch.int64, device=dev)
    kc, ep = _key(key, num_worlds, dev)
    _check(nat.lib().dk_dr_randomize_params(num_worlds, len(names), _ptr(nom), len(ranges),
                                            _ptr(fld), _ptr(dst), _ptr(lo_t), _ptr(hi_t),
                                            ctypes.byref(kc), _ptr(out), _ptr(fail),
                                            _stream(dev)))
    f = int(fail.item())
    if f != -1:
        raise ConfigError(f"could not draw a physical value for {ranges[f % len(ranges)].path!r}")
    return out, names


class DelayLineBatch:
    """``num_worlds`` DelayLines (randomization.py:27-62) of ``dim``-vectors on
    the GPU: a [num_worlds, max_delay + 1, dim] ring per batch.  ``reset(key)``
    draws each world's episode delay (Generator.integers(min, max + 1) from its
    stream); ``push_pop(value, key)`` appends and returns the aged values (a
    fresh per-step delay from ``key`` when ``per_step``)."""

    def __init__(self, num_worlds: int, dim: int, min_delay: int, max_delay: int,
                 per_step: bool = False, dtype=None, device=None):
        torch = _torch()
        if min_delay < 0 or max_delay < min_delay:
            raise ConfigError("delay bounds must satisfy 0 <= min <= max")
        self.num_worlds, self.dim = int(num_worlds), int(dim)
        self.min_delay, self.max_delay, self.per_step = int(min_delay), int(max_delay), per_step
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        self.device = dev
        self.dtype = dtype or torch.float32
        self.ring = torch.zeros((self.num_worlds, max_delay + 1, dim), dtype=self.dtype,
                                device=dev)
        self.head = torch.zeros(self.num_worlds, dtype=torch.int32, device=dev)
        self.count = torch.zeros_like(self.head)
        self.delay = torch.zeros_like(self.head)
        self._has_delay = False

    def reset(self, key: NoiseKey):
        kc, ep = _key(key, self.num_worlds, self.device)
        _check(nat.lib().dk_dr_delay_reset(self.num_worlds, self.min_delay, self.max_delay,
                                           ctypes.byref(kc), _ptr(self.delay), _ptr(self.count),
                                           _ptr(self.head), _stream(self.device)))
        self._has_delay = True

    def push_pop(self, value, key: NoiseKey | None = None):
        if not self.per_step and not self._has_delay:
            raise ConfigError("delay line used before reset")
        if self.per_step and key is None:
            raise ConfigError("per-step delay lines need a key per push_pop")
        v = value.to(self.dtype).reshape(self.num_worlds, self.dim).contiguous()
        out = _torch().empty_like(v)
        kc, ep = _key(key or NoiseKey(), self.num_worlds, self.device)
        _check(nat.lib().dk_dr_delay_push_pop(_dtype_code(v), self.num_worlds, self.dim,
                                              self.min_delay, self.max_delay, int(self.per_step),
                                              _ptr(self.ring), _ptr(self.head), _ptr(self.count),
                                              _ptr(self.delay), ctypes.byref(kc), _ptr(v),
                                              _ptr(out), _stream(self.device)))
        return out.reshape(value.shape)


def pose_injection_batch(pose, prob: float, bounds, key: NoiseKey):
    """randomization.pose_injection per row: returns (pose, injected mask)."""
    torch = _torch()
    if not 0.0 <= prob <= 1.0:
        raise InvalidInputError("prob must lie in [0, 1]")
    p = pose.contiguous().clone()
    n, dim = p.shape
    b = torch.as_tensor(np.asarray(bounds, dtype=np.float64), device=p.device).contiguous()
    inj = torch.empty(n, dtype=torch.uint8, device=p.device)
    kc, ep = _key(key, n, p.device)
    _check(nat.lib().dk_dr_pose_injection(_dtype_code(p), n, dim, _ptr(p), _ptr(b), float(prob),
                                          ctypes.byref(kc), _ptr(inj), _stream(p.device)))
    return p, inj.bool()


def curriculum_update_batch(state, success, max_level: int = 10, promotion_threshold: int = 1):
    """curriculum_update on [n, 4] int64 (level, successes_at_level, episodes,
    total_successes); returns the new state tensor."""
    torch = _torch()
    st = state.to(torch.int64).contiguous().clone()
    s = success.to(torch.uint8).contiguous()
    _check(nat.lib().dk_dr_curriculum(st.shape[0], _ptr(st), _ptr(s), int(max_level),
                                      int(promotion_threshold), _stream(st.device)))
    return st


__all__ = [
    "DelayLineBatch", "NoiseKey", "ObservationNoise", "PDParams", "RewardBreakdownBatch",
    "RewardTermConfig", "TERM_NAMES", "advance_phase_batch", "apply_sensor_noise_batch",
    "build_locomotion_observation_batch", "curriculum_update_batch", "frames_from_reference",
    "locomotion_tail", "pd_batch", "pose_injection_batch", "progress_clip_reward_batch",
    "randomize_params_batch", "total_reward_batch",
]
