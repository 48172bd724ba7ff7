"""Batched articulated contact physics on B200.

``DevicePhysics`` steps N Go1-shaped worlds in lockstep through the sm_100a
kernel in csrc/physics.cuh (one lane quad per world, lane = limb), behind the
C ABI ``dk_phys_*`` (include/deskrl_b200.h).  State is MuJoCo-shaped:
``qpos`` [N, 19] (trunk pos, trunk quat w-x-y-z, 12 joints) and ``qvel``
[N, 18] (trunk linear velocity in the world frame, angular velocity in the
trunk frame, 12 joint velocities); ``ctrl`` [N, 12] are joint position
targets of the PD actuators.  ``step`` returns the last step's diagnostics
(``qacc``, ``qfrc_bias``, ``qfrc_constraint``, ``act_force``, ``ncon``,
``contact_geom`` pairs, ``contact_dist`` / ``pos`` / ``force``,
``solver_iter``, ``sensordata``) as CUDA tensors.

The reference has no articulated physics (SPEC.md:8 puts the MJX/MuJoCo solver
out of scope); parity is against oracle/physics.c and is UNPINNED.  There is
no CPU fallback: without the library or a GPU this raises.
"""

from __future__ import annotations

import ctypes

from . import _native as nat
from .envkit import _ERR, BackendError, ConfigError, InvalidInputError, _check  # noqa: F401
from .physmodel import MAXCON, NQ, NSENSOR, NU, NV, PhysModel, PhysModelC, go1_model, home_qpos


def default_model_c() -> PhysModelC:
    """The library's built-in Go1-shaped model (dk_phys_default_model)."""
    m = PhysModelC()
    _check(nat.lib().dk_phys_default_model(ctypes.byref(m)))
    return m


class _DiagC(ctypes.Structure):
    _fields_ = [(f, ctypes.c_void_p) for f in (
        "qacc", "qfrc_bias", "qfrc_constraint", "act_force", "ncon", "contact_geom",
        "contact_dist", "contact_pos", "contact_force", "solver_iter", "sensordata")]


DIAG_FIELDS = tuple(f for f, _ in _DiagC._fields_)


class DevicePhysics:
    """N worlds of the articulated model on one GPU (CUDA tensors in/out,
    enqueued on the current stream)."""

    def __init__(self, model: PhysModel | None = None, num_worlds: int = 1, dtype="float32",
                 device: int | None = None):
        import torch

        self._torch = torch
        self.model = (model or go1_model()).validate()
        self.num_worlds = int(num_worlds)
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
        self._mc = self.model.to_c()
        h = ctypes.c_void_p()
        _check(self._lib.dk_phys_create(ctypes.byref(self._mc), code, self.num_worlds,
                                        int(device), ctypes.byref(h)))
        self.h = h

    def _stream(self):
        return ctypes.c_void_p(self._torch.cuda.current_stream(self.device).cuda_stream)

    def _t(self, x, shape, name):
        torch = self._torch
        t = torch.as_tensor(x, device=self.device, dtype=self.dtype)
        if tuple(t.shape) != shape:
            raise InvalidInputError(f"{name} must have shape {shape}, got {tuple(t.shape)}")
        return t.contiguous()

    def set_state(self, qpos=None, qvel=None):
        n = self.num_worlds
        qp = None if qpos is None else self._t(qpos, (n, NQ), "qpos")
        qv = None if qvel is None else self._t(qvel, (n, NV), "qvel")
        _check(self._lib.dk_phys_set_state(self.h, None if qp is None else qp.data_ptr(),
                                           None if qv is None else qv.data_ptr(),
                                           self._stream()))
        self._keep = (qp, qv)  # alive until the transpose has run (stream-ordered)

    def reset(self, qpos=None, qvel=None):
        """Home keyframe (or the given state) for every world, zero velocity."""
        torch = self._torch
        n = self.num_worlds
        qp = torch.as_tensor(home_qpos(n) if qpos is None else qpos, dtype=self.dtype,
                             device=self.device)
        qv = torch.zeros((n, NV), dtype=self.dtype, device=self.device) if qvel is None else qvel
        self.set_state(qp, qv)

    def state(self):
        torch = self._torch
        n = self.num_worlds
        qp = torch.empty((n, NQ), dtype=self.dtype, device=self.device)
        qv = torch.empty((n, NV), dtype=self.dtype, device=self.device)
        _check(self._lib.dk_phys_get_state(self.h, qp.data_ptr(), qv.data_ptr(), self._stream()))
        return qp, qv

    def alloc_diag(self):
        torch = self._torch
        n, dt, dev = self.num_worlds, self.dtype, self.device
        i32 = torch.int32
        return {"qacc": torch.empty((n, NV), dtype=dt, device=dev),
                "qfrc_bias": torch.empty((n, NV), dtype=dt, device=dev),
                "qfrc_constraint": torch.empty((n, NV), dtype=dt, device=dev),
                "act_force": torch.empty((n, NU), dtype=dt, device=dev),
                "ncon": torch.empty((n,), dtype=i32, device=dev),
                "contact_geom": torch.empty((n, MAXCON, 2), dtype=i32, device=dev),
                "contact_dist": torch.empty((n, MAXCON), dtype=dt, device=dev),
                "contact_pos": torch.empty((n, MAXCON, 3), dtype=dt, device=dev),
                "contact_force": torch.empty((n, MAXCON, 3), dtype=dt, device=dev),
                "solver_iter": torch.empty((n,), dtype=i32, device=dev),
                "sensordata": torch.empty((n, NSENSOR), dtype=dt, device=dev)}

    def step(self, ctrl, num_steps: int = 1, diag: bool | dict = True):
        """Advance every world ``num_steps`` physics steps with ``ctrl`` [N, 12]
        held.  Returns the diagnostics dict of the last step (or None)."""
        c = self._t(ctrl, (self.num_worlds, NU), "ctrl")
        out = None
        dptr = None
        if diag is not False and diag is not None:
            out = diag if isinstance(diag, dict) else self.alloc_diag()
            d = _DiagC(*[out[f].data_ptr() if out.get(f) is not None else None
                         for f in DIAG_FIELDS])
            dptr = ctypes.byref(d)
        _check(self._lib.dk_phys_step(self.h, int(num_steps), c.data_ptr(), dptr,
                                      self._stream()))
        self._keep_ctrl = c
        return out

    def inspect(self):
        """G1 quantities at the current state: M [N, 18, 18] (armature, no
        implicit-damping term), qfrc_bias [N, 18], xpos / xipos [N, 13, 3]."""
        torch = self._torch
        n, dt, dev = self.num_worlds, self.dtype, self.device
        out = {"M": torch.empty((n, NV, NV), dtype=dt, device=dev),
               "qfrc_bias": torch.empty((n, NV), dtype=dt, device=dev),
               "xpos": torch.empty((n, 13, 3), dtype=dt, device=dev),
               "xipos": torch.empty((n, 13, 3), dtype=dt, device=dev)}
        _check(self._lib.dk_phys_inspect(self.h, out["M"].data_ptr(),
                                         out["qfrc_bias"].data_ptr(), out["xpos"].data_ptr(),
                                         out["xipos"].data_ptr(), self._stream()))
        return out

    def check(self):
        """Synchronise; raise InvalidInputError if a step met a non-SPD matrix."""
        self._torch.cuda.current_stream(self.device).synchronize()
        _check(self._lib.dk_phys_check(self.h))

    @property
    def kernel_launches(self) -> int:
        return int(self._lib.dk_phys_kernel_launches(self.h))

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self._lib.dk_phys_destroy(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


__all__ = ["DIAG_FIELDS", "DevicePhysics", "default_model_c"]
