"""Batched env step on B200: drop-in ``BatchEnv`` plus a device-resident API.

Mirrors the reference's env runtime (deskrl ``envkit``,
/root/reference/pkg/src/deskrl/envkit.py): the same configuration dataclasses
(``EnvConfig`` envkit.py:56-75, ``DynamicsParams`` dynamics.py:36-72), the same
task ids (``registered_tasks`` envkit.py:461-462), the same ``BatchEnv``
surface (envkit.py:595-650: ``reset(seed)``, ``step(actions, autoreset)``,
``close()``, ``num_envs``, ``action_dim``, ``config``, ``envs``) and the same
error classes and messages.  All stepping runs in the sm_100a kernels of
libdeskrl_b200.so through the C ABI of include/deskrl_b200.h; there is no
CPU fallback.

Two front-ends:

* ``BatchEnv`` -- numpy in / numpy out, synchronous, exactly the reference's
  return types (float64 observations, ``infos`` list of dicts with the reward
  terms and ``terminal_observation``).  Pass ``dtype="float32"`` to compute in
  float32.
* ``DeviceBatchEnv`` -- torch CUDA tensors in / out, asynchronous on the
  current stream, plus ``rollout(actions[K, N, A])`` that fuses K steps into
  one kernel.  Worlds can be sharded across GPUs with ``env_index_offset``.
"""

from __future__ import annotations

import ctypes
from collections.abc import Sequence
from dataclasses import dataclass, field, replace

import numpy as np

from . import _native as nat


# ---------------------------------------------------------------------------
# errors (same names, bases and messages as the reference)


class ConfigError(ValueError):
    """Malformed configuration (reference: randomization.py:19)."""


class InvalidInputError(ValueError):
    """Out-of-contract input (reference: mathcore.py:22)."""


class UsageError(RuntimeError):
    """Env API driven out of contract (reference: envkit.py:37)."""


class BackendError(RuntimeError):
    """CUDA / driver failure inside the B200 backend."""


_ERR = {
    nat.DK_ERR_CONFIG: ConfigError,
    nat.DK_ERR_INVALID_INPUT: InvalidInputError,
    nat.DK_ERR_USAGE: UsageError,
    nat.DK_ERR_CUDA: BackendError,
}


def _check(rc: int) -> None:
    if rc != nat.DK_OK:
        raise _ERR.get(rc, BackendError)(nat.last_error())


# ---------------------------------------------------------------------------
# configuration (mirrors of the reference dataclasses)


@dataclass(frozen=True)
class DynamicsParams:
    """Physical constants (reference: dynamics.py:36-72)."""

    dt: float = 0.01
    gravity: float = 9.81
    pend_mass: float = 1.0
    pend_length: float = 0.5
    pend_damping: float = 0.05
    pend_torque_limit: float = 2.5
    cart_mass: float = 1.0
    pole_mass: float = 0.1
    pole_length: float = 0.5
    rail_limit: float = 1.8
    cart_force_limit: float = 10.0
    link1_mass: float = 1.0
    link2_mass: float = 1.0
    link1_length: float = 1.0
    link2_length: float = 1.0
    link_damping: float = 0.0
    elbow_torque_limit: float = 8.0
    reacher_torque_limit: float = 1.0

    def __post_init__(self):
        if self.dt <= 0:
            raise InvalidInputError("dt must be positive")
        for name in ("pend_mass", "pend_length", "cart_mass", "pole_mass", "pole_length",
                     "link1_mass", "link2_mass", "link1_length", "link2_length"):
            if getattr(self, name) <= 0:
                raise InvalidInputError(f"{name} must be positive")

    def with_dt(self, dt: float) -> "DynamicsParams":
        return replace(self, dt=dt)


@dataclass(frozen=True)
class EnvConfig:
    """Env configuration (reference: envkit.py:56-75)."""

    task: str = "cartpole-balance"
    episode_length: int = 1000
    action_repeat: int = 1
    dt: float | None = None
    obs_mode: str = "state"
    seed: int = 0
    image_size: int = 64
    visual_randomization: bool = False
    wide_init: bool = False
    randomization: object = None  # accepted, unused -- as in the reference

    def __post_init__(self):
        if self.episode_length <= 0:
            raise ConfigError("episode_length must be positive")
        if self.action_repeat < 1:
            raise ConfigError("action_repeat must be >= 1")
        if self.obs_mode not in ("state", "pixels"):
            raise ConfigError(f"unknown obs_mode {self.obs_mode!r}")


@dataclass(frozen=True)
class TaskSpec:
    """What the reference exposes as ``Environment.task`` (envkit.py:224-252)."""

    id: str
    index: int
    action_dim: int
    obs_dim: int
    state_dim: int
    default_dt: float
    info_keys: tuple
    params: DynamicsParams = field(default_factory=DynamicsParams)
    pixels: bool = False              # cartpole-balance-pixels / obs_mode "pixels"
    image_size: int = 64
    visual_randomization: bool = False


_TASK_TABLE = {
    # id: (abi index, action_dim, obs_dim, state_dim, default_dt, info keys)
    "pendulum-swingup": (0, 1, 3, 2, 0.01, ("upright",)),
    "cartpole-balance": (1, 1, 5, 4, 0.01, ("upright", "centered", "still")),
    "acrobot-swingup": (2, 1, 6, 4, 0.01, ("tip_height",)),
    "reacher-easy": (3, 2, 10, 4, 0.005, ("distance",)),
}


def registered_tasks() -> list[str]:
    """Task ids, identical to the reference's registry (envkit.py:461-462)."""
    return sorted(_TASK_TABLE) + ["cartpole-balance-pixels"]


def resolve_task(config, params=None) -> TaskSpec:
    """Validate ``config`` like Environment.__init__ (envkit.py:474-487)."""
    name = config.task
    pixels = getattr(config, "obs_mode", "state") == "pixels" or name.endswith("-pixels")
    if name.endswith("-pixels"):
        base = name[: -len("-pixels")]
        if base != "cartpole-balance":
            raise ConfigError(f"no pixel variant for task {base!r}")
        name = base
    if name not in _TASK_TABLE:
        raise ConfigError(f"unknown task id {config.task!r}")
    if pixels and name != "cartpole-balance":
        raise ConfigError(f"no pixel variant for task {name!r}")
    idx, a, o, s, default_dt, keys = _TASK_TABLE[name]
    base_params = params or DynamicsParams()
    dt = config.dt if config.dt is not None else default_dt
    p = DynamicsParams(**{f: float(getattr(base_params, f)) for f in nat.PARAM_FIELDS})
    return TaskSpec(name, idx, a, o, s, default_dt, keys, p.with_dt(float(dt)), pixels,
                    int(getattr(config, "image_size", 64)),
                    bool(getattr(config, "visual_randomization", False)))


def _pixel_obs(spec, num_envs, seed, env_index_offset, dtype, device):
    """PixelObservation for a pixel task (pixelrender via paper_2502_08844_b200.pixels)."""
    from .pixels import PixelObservation

    return PixelObservation(num_envs, spec.image_size, spec.visual_randomization, seed,
                            env_index_offset, spec.params.pole_length, dtype, device)


def _dtype_code(dtype) -> int:
    name = getattr(dtype, "name", None) or str(dtype)
    name = name.replace("torch.", "")
    if name in ("float32", "f32", "float"):
        return nat.DK_F32
    if name in ("float64", "f64", "double"):
        return nat.DK_F64
    raise ConfigError(f"unsupported dtype {dtype!r} (float32 or float64)")


class _Handle:
    """Owns one dk_env handle."""

    def __init__(self, config, num_envs: int, params, dtype, device_index: int,
                 env_index_offset: int):
        if num_envs < 1:
            raise ConfigError("num_envs and num_workers must be >= 1")
        self.spec = resolve_task(config, params)
        self.dtype_code = _dtype_code(dtype)
        self.np_dtype = np.float64 if self.dtype_code == nat.DK_F64 else np.float32
        self.num_envs = int(num_envs)
        self.device_index = int(device_index)
        self.env_index_offset = int(env_index_offset)
        self._lib = nat.lib()
        self._cfg = nat.EnvConfigC(self.spec.index, self.dtype_code, int(config.episode_length),
                                   int(config.action_repeat), int(bool(config.wide_init)), 0,
                                   int(config.seed) & (2**64 - 1))
        p = self.spec.params
        self._params = nat.DynamicsParamsC(*[float(getattr(p, f)) for f in nat.PARAM_FIELDS])
        h = ctypes.c_void_p()
        _check(self._lib.dk_env_create(ctypes.byref(self._cfg), ctypes.byref(self._params),
                                       self.num_envs, self.env_index_offset, self.device_index,
                                       ctypes.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self._lib.dk_env_destroy(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def get_state(self):
        n = self.num_envs
        s = np.zeros((n, 4))
        t = np.zeros((n, 2))
        steps = np.zeros(n, dtype=np.int64)
        ep = np.zeros(n, dtype=np.int64)
        nr = np.zeros(n, dtype=np.uint8)
        _check(self._lib.dk_env_get_state(self.h, s.ctypes.data, t.ctypes.data, steps.ctypes.data,
                                          ep.ctypes.data, nr.ctypes.data))
        return s, t, steps, ep, nr.astype(bool)

    def set_state(self, state=None, target=None, steps=None, episode=None, needs_reset=None):
        def arr(x, dt, shape):
            return None if x is None else np.ascontiguousarray(np.asarray(x, dtype=dt).reshape(shape))

        n = self.num_envs
        s = arr(state, np.float64, (n, 4))
        t = arr(target, np.float64, (n, 2))
        st = arr(steps, np.int64, (n,))
        ep = arr(episode, np.int64, (n,))
        nr = arr(needs_reset, np.uint8, (n,))
        ptr = lambda a: None if a is None else a.ctypes.data  # noqa: E731
        _check(self._lib.dk_env_set_state(self.h, ptr(s), ptr(t), ptr(st), ptr(ep), ptr(nr)))

    @property
    def kernel_launches(self) -> int:
        return int(self._lib.dk_env_kernel_launches(self.h))


# ---------------------------------------------------------------------------
# drop-in BatchEnv (numpy)


class _Infos(Sequence):
    """``infos`` of BatchEnv.step: list-like of per-world dicts, built lazily.

    infos[i] holds the reward terms of world i (envkit.py:289-453) and, when
    the world auto-reset, ``terminal_observation`` (envkit.py:632-634)."""

    def __init__(self, keys, info, term_mask, term_obs, term_pixels=None):
        self._keys = keys
        self._info = info
        self._mask = term_mask
        self._term = term_obs
        self._term_pixels = term_pixels
        self._built = {}  # index -> dict: persistent like the reference's list of dicts

    def __len__(self):
        return self._info.shape[0]

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        if i < 0:
            i += len(self)
        if not 0 <= i < len(self):
            raise IndexError(i)
        d = self._built.get(i)
        if d is not None:
            return d
        d = self._built[i] = {k: float(self._info[i, j]) for j, k in enumerate(self._keys)}
        if self._mask is not None and self._mask[i]:
            t = np.array(self._term[i], dtype=np.float64)
            d["terminal_observation"] = {"state": t, "privileged_state": t.copy()}
            if self._term_pixels is not None:
                d["terminal_observation"]["pixels"] = self._term_pixels[i]
        return d


class _EnvView:
    """Read-mostly view of one world, standing in for deskrl ``Environment``
    objects in ``BatchEnv.envs`` (envkit.py:605; used by serve.py:62 and
    cli.py:436-441)."""

    def __init__(self, owner: "BatchEnv", index: int):
        self._owner = owner
        self.env_index = owner.env_index_offset + index
        self._i = index
        self.task = owner._h.spec
        self.action_dim = owner.action_dim
        self.config = owner.config

    def _row(self):
        s, t, steps, ep, nr = self._owner._state_snapshot()
        return s[self._i], t[self._i], steps[self._i], ep[self._i], nr[self._i]

    @property
    def state(self):
        s, *_ = self._row()
        return tuple(float(v) for v in s[: self.task.state_dim])

    @property
    def steps(self):
        return int(self._row()[2])

    @property
    def _episode(self):
        return int(self._row()[3])

    @property
    def _needs_reset(self):
        return bool(self._row()[4])

    @property
    def _target(self):
        if self.task.id != "reacher-easy" or self._needs_reset and self._episode < 0:
            return None
        return np.array(self._row()[1])

    def observation_shapes(self) -> dict:
        o = self.task.obs_dim
        shapes = {"state": (o,), "privileged_state": (o,)}
        if getattr(self.task, "pixels", False):
            shapes["pixels"] = (self.task.image_size, self.task.image_size, 3)
        return shapes


class BatchEnv:
    """N worlds stepped together on one B200 (reference: envkit.py:595-650).

    Same constructor and methods as the reference; ``num_workers`` is
    accepted for compatibility (results never depend on it).
    Keyword-only extras: ``dtype`` ("float64" default -- the reference's
    arithmetic type -- or "float32"), ``device`` (CUDA index) and
    ``env_index_offset`` (global index of world 0 for sharding).
    """

    def __init__(self, config, num_envs: int, num_workers: int = 1, params=None, *,
                 dtype="float64", device: int | None = None, env_index_offset: int = 0):
        if num_envs < 1 or num_workers < 1:
            raise ConfigError("num_envs and num_workers must be >= 1")
        self.config = config
        self.num_envs = int(num_envs)
        self.num_workers = int(num_workers)
        self.env_index_offset = int(env_index_offset)
        if device is None:
            device = _current_device()
        self._h = _Handle(config, num_envs, params, dtype, device, env_index_offset)
        spec = self._h.spec
        self.action_dim = spec.action_dim
        self.obs_dim = spec.obs_dim
        self.dtype = np.dtype(self._h.np_dtype)
        self._alloc_host_buffers()
        self._envs = None
        self._version, self._snap = 0, None
        self._pix = None
        if spec.pixels:  # rendered on the device from the state observations
            import torch

            self._torch = torch
            self._pix_dev = torch.device("cuda", device)
            self._pix = _pixel_obs(spec, self.num_envs, int(config.seed), self.env_index_offset,
                                   torch.float64, self._pix_dev)

    # pinned host staging (allocated once; outputs are copied out per call)
    def _alloc_host_buffers(self):
        n, o, a, i = self.num_envs, self.obs_dim, self.action_dim, len(self._h.spec.info_keys)
        dt = self._h.np_dtype
        self._b_act = _pinned((n, a), dt)
        self._b_obs = _pinned((n, o), dt)
        self._b_rew = _pinned((n,), dt)
        self._b_done = _pinned((n,), np.uint8)
        self._b_trunc = _pinned((n,), np.uint8)
        self._b_term = _pinned((n, o), dt)
        self._b_mask = _pinned((n,), np.uint8)
        self._b_info = _pinned((n, i), dt)

    def _state_snapshot(self):
        """One device->host copy of every world's state per env version
        (invalidated by reset / step), shared by all ``envs[i]`` views, so
        walking ``envs`` is O(N), not O(N^2)."""
        if self._snap is None or self._snap[0] != self._version:
            self._snap = (self._version, self._h.get_state())
        return self._snap[1]

    @property
    def envs(self):
        if self._envs is None:
            self._envs = [_EnvView(self, i) for i in range(self.num_envs)]
        return self._envs

    def reset(self, seed: int | None = None) -> dict:
        if seed is not None:
            self.config = _replace_seed(self.config, seed)
            if self._envs is not None:
                for e in self._envs:
                    e.config = self.config
        self._version += 1
        _check(self._h._lib.dk_env_reset_host(self._h.h, int(seed is not None),
                                              0 if seed is None else int(seed) & (2**64 - 1),
                                              self._b_obs.ctypes.data))
        obs = self._b_obs.astype(np.float64)
        out = {"state": obs, "privileged_state": obs.copy()}
        if self._pix is not None:
            t = self._torch.as_tensor(obs, device=self._pix_dev)
            out["pixels"] = self._pix.reset(t, seed).cpu().numpy()
        return out

    def step(self, actions, autoreset: bool = True):
        actions = np.asarray(actions, dtype=float)
        if actions.shape[0] != self.num_envs:
            raise InvalidInputError("actions batch size mismatch")
        a = actions.reshape(self.num_envs, self.action_dim)
        if self._h.dtype_code == nat.DK_F32:
            # clip before narrowing so a huge finite action clips like the
            # reference instead of overflowing to inf; NaN/inf still trip the
            # device-side check
            a = np.where(np.isfinite(a), np.clip(a, -1.0, 1.0), a)
        np.copyto(self._b_act, a, casting="unsafe")
        self._version += 1
        _check(self._h._lib.dk_env_step_host(
            self._h.h, self._b_act.ctypes.data, int(bool(autoreset)), self._b_obs.ctypes.data,
            self._b_rew.ctypes.data, self._b_done.ctypes.data, self._b_trunc.ctypes.data,
            self._b_term.ctypes.data, self._b_mask.ctypes.data, self._b_info.ctypes.data))
        obs = self._b_obs.astype(np.float64)
        rewards = self._b_rew.astype(np.float64)
        dones = self._b_done.astype(bool)
        truncs = self._b_trunc.astype(bool)
        mask = self._b_mask.astype(bool)
        term = self._b_term.astype(np.float64) if mask.any() else None
        out = {"state": obs, "privileged_state": obs.copy()}
        term_pix = None
        if self._pix is not None:
            tt = self._torch
            d = self._pix_dev
            so = {"obs": tt.as_tensor(obs, device=d),
                  "terminal_obs": tt.as_tensor(self._b_term.astype(np.float64), device=d),
                  "terminal_mask": tt.as_tensor(self._b_mask.astype(bool), device=d)}
            pix, tp = self._pix.step(so, terminal=term is not None)
            out["pixels"] = pix.cpu().numpy()
            term_pix = tp.cpu().numpy() if tp is not None else None
        infos = _Infos(self._h.spec.info_keys, self._b_info.astype(np.float64),
                       mask if term is not None else None, term, term_pix)
        return out, rewards, dones, truncs, infos

    def close(self):
        self._h.close()

    @property
    def kernel_launches(self) -> int:
        return self._h.kernel_launches


# ---------------------------------------------------------------------------
# device-resident API (torch CUDA tensors)


class DeviceBatchEnv:
    """Device-resident batched env: CUDA tensors in and out, asynchronous.

    ``step`` / ``rollout`` enqueue on the current torch stream.  Validation is
    batch-atomic on the device; an invalid call leaves the worlds untouched
    and raises at the next ``check()`` (or ``reset``/``state``), like an
    asynchronous CUDA error.
    """

    def __init__(self, config, num_envs: int, params=None, *, dtype="float32", device=None,
                 env_index_offset: int = 0):
        import torch

        self._torch = torch
        dev = torch.device("cuda", _current_device() if device is None else
                           (device if isinstance(device, int) else torch.device(device).index or 0))
        self.device = dev
        self.config = config
        self.num_envs = int(num_envs)
        self.env_index_offset = int(env_index_offset)
        self._h = _Handle(config, num_envs, params, dtype, dev.index, env_index_offset)
        self.spec = self._h.spec
        self.action_dim = self.spec.action_dim
        self.obs_dim = self.spec.obs_dim
        self.info_keys = self.spec.info_keys
        self.dtype = torch.float64 if self._h.dtype_code == nat.DK_F64 else torch.float32
        self._pix = (_pixel_obs(self.spec, self.num_envs, int(config.seed), self.env_index_offset,
                                self.dtype, dev) if self.spec.pixels else None)

    def _stream(self):
        return ctypes.c_void_p(self._torch.cuda.current_stream(self.device).cuda_stream)

    @staticmethod
    def _ptr(t):
        return None if t is None else ctypes.c_void_p(t.data_ptr())

    def reset(self, seed: int | None = None):
        self.check()
        if seed is not None:
            self.config = _replace_seed(self.config, seed)
        obs = self._torch.empty((self.num_envs, self.obs_dim), dtype=self.dtype,
                                device=self.device)
        _check(self._h._lib.dk_env_reset(self._h.h, int(seed is not None),
                                         0 if seed is None else int(seed) & (2**64 - 1),
                                         self._ptr(obs), self._stream()))
        out = {"state": obs, "privileged_state": obs}
        if self._pix is not None:
            out["pixels"] = self._pix.reset(obs, seed)
        return out

    def _outputs(self, lead, with_info):
        t, d, n, o = self._torch, self.device, self.num_envs, self.obs_dim
        return dict(
            obs=t.empty((*lead, n, o), dtype=self.dtype, device=d),
            reward=t.empty((*lead, n), dtype=self.dtype, device=d),
            done=t.empty((*lead, n), dtype=t.bool, device=d),
            trunc=t.empty((*lead, n), dtype=t.bool, device=d),
            terminal_obs=t.empty((*lead, n, o), dtype=self.dtype, device=d),
            terminal_mask=t.empty((*lead, n), dtype=t.bool, device=d),
            info=(t.empty((*lead, n, len(self.info_keys)), dtype=self.dtype, device=d)
                  if with_info else None),
        )

    def _check_actions(self, actions, lead):
        if not actions.is_cuda or actions.device != self.device:
            raise InvalidInputError(f"actions must be a CUDA tensor on {self.device}")
        want = (*lead, self.num_envs, self.action_dim)
        if actions.dim() == len(want) - 1 and self.action_dim == 1:
            actions = actions.unsqueeze(-1)
        if tuple(actions.shape[: len(lead) + 1]) != (*lead, self.num_envs):
            raise InvalidInputError("actions batch size mismatch")
        if tuple(actions.shape) != want:
            raise InvalidInputError(f"actions must have shape {want}")
        if actions.dtype != self.dtype:
            actions = actions.to(self.dtype)
        return actions.contiguous()

    def step(self, actions, autoreset: bool = True, with_info: bool = True, out: dict | None = None):
        a = self._check_actions(actions, ())
        o = out or self._outputs((), with_info)
        _check(self._h._lib.dk_env_step(
            self._h.h, self._ptr(a), int(bool(autoreset)), self._ptr(o["obs"]),
            self._ptr(o["reward"]), self._ptr(o["done"]), self._ptr(o["trunc"]),
            self._ptr(o["terminal_obs"]), self._ptr(o["terminal_mask"]), self._ptr(o["info"]),
            self._stream()))
        if self._pix is not None:  # obs["pixels"] of cartpole-balance-pixels (envkit.py:561-576)
            o["pixels"], o["terminal_pixels"] = self._pix.step(o)
        return o

    def rollout(self, actions, with_info: bool = False, out: dict | None = None):
        """K fused autoreset steps; actions [K, N, A] -> outputs [K, N, ...]."""
        if self._pix is not None:
            raise ConfigError("pixel observations are rendered per step: use step()")
        if actions.dim() < 2:
            raise InvalidInputError("rollout actions must be [K, N, A]")
        K = int(actions.shape[0])
        a = self._check_actions(actions, (K,))
        o = out or self._outputs((K,), with_info)
        _check(self._h._lib.dk_env_rollout(
            self._h.h, K, self._ptr(a), self._ptr(o["obs"]), self._ptr(o["reward"]),
            self._ptr(o["done"]), self._ptr(o["trunc"]), self._ptr(o["terminal_obs"]),
            self._ptr(o["terminal_mask"]), self._ptr(o.get("info")), self._stream()))
        return o

    def check(self):
        """Synchronise and raise the first pending step error, if any."""
        k = ctypes.c_int64(0)
        i = ctypes.c_int64(0)
        rc = self._h._lib.dk_env_check_error(self._h.h, self._stream(), ctypes.byref(k),
                                             ctypes.byref(i))
        if rc != nat.DK_OK:
            err = _ERR.get(rc, BackendError)(nat.last_error())
            err.step_index, err.env_index = int(k.value), int(i.value)
            raise err

    def state(self):
        """(state [N,4], target [N,2], steps, episode, needs_reset) as numpy."""
        self.check()
        return self._h.get_state()

    def set_state(self, **kw):
        self._torch.cuda.current_stream(self.device).synchronize()
        self._h.set_state(**kw)

    def close(self):
        self._h.close()

    @property
    def kernel_launches(self) -> int:
        return self._h.kernel_launches


# ---------------------------------------------------------------------------
# helpers


def _current_device() -> int:
    try:
        import torch

        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except Exception:
        pass
    return 0


def _pinned(shape, dtype):
    """Page-locked numpy buffer (torch allocator; falls back to pageable)."""
    try:
        import torch

        if torch.cuda.is_available():
            tdt = {np.float32: torch.float32, np.float64: torch.float64,
                   np.uint8: torch.uint8}[np.dtype(dtype).type]
            return torch.empty(shape, dtype=tdt, pin_memory=True).numpy()
    except Exception:
        pass
    return np.empty(shape, dtype=dtype)


def _replace_seed(config, seed):
    try:
        return replace(config, seed=seed)
    except TypeError:
        config.seed = seed
        return config


@dataclass
class StepResult:
    """Result of Environment.step (reference: envkit.py:78-84)."""

    observation: dict
    reward: float
    done: bool
    truncated: bool
    info: dict = field(default_factory=dict)


class Environment:
    """A single world (reference: envkit.py:469-584) on the B200 backend.

    Same lifecycle as the reference: ``reset(seed=None) -> obs``,
    ``step(action) -> StepResult`` (no autoreset: stepping past truncation
    raises ``UsageError``), ``observation_shapes()``, ``state``, ``steps``.
    ``env_index`` keys the world's Philox stream like the reference's."""

    def __init__(self, config, env_index: int = 0, params=None, *, dtype="float64",
                 device: int | None = None):
        self.config = config
        self.env_index = int(env_index)
        self._b = BatchEnv(config, 1, params=params, dtype=dtype, device=device,
                           env_index_offset=env_index)
        self.task = self._b._h.spec
        self.action_dim = self.task.action_dim

    def reset(self, seed: int | None = None) -> dict:
        o = self._b.reset(seed)
        self.config = self._b.config
        return {k: v[0] for k, v in o.items()}

    def step(self, action) -> StepResult:
        a = np.asarray(action, dtype=float).reshape(1, self.action_dim)
        obs, r, d, t, infos = self._b.step(a, autoreset=False)
        info = dict(infos[0])
        return StepResult({k: v[0] for k, v in obs.items()}, float(r[0]), bool(d[0]),
                          bool(t[0]), info)

    @property
    def state(self):
        return self._b.envs[0].state

    @property
    def steps(self):
        return self._b.envs[0].steps

    def observation_shapes(self) -> dict:
        o = self.task.obs_dim
        shapes = {"state": (o,), "privileged_state": (o,)}
        if getattr(self.task, "pixels", False):
            shapes["pixels"] = (self.task.image_size, self.task.image_size, 3)
        return shapes

    def close(self):
        self._b.close()


def make_env(task: str, **kwargs) -> Environment:
    """Single-world env (reference: envkit.py:587-588)."""
    dtype = kwargs.pop("dtype", "float64")
    return Environment(EnvConfig(task=task, **kwargs), dtype=dtype)


def make_batch_env(task: str, num_envs: int, **kwargs) -> BatchEnv:
    """BatchEnv of ``num_envs`` worlds of ``task`` (cf. make_env, envkit.py:587-588)."""
    dtype = kwargs.pop("dtype", "float64")
    return BatchEnv(EnvConfig(task=task, **kwargs), num_envs, dtype=dtype)


__all__ = [
    "BackendError", "BatchEnv", "ConfigError", "DeviceBatchEnv", "DynamicsParams", "EnvConfig",
    "Environment", "StepResult", "make_env",
    "InvalidInputError", "TaskSpec", "UsageError", "make_batch_env", "registered_tasks",
    "resolve_task",
]
