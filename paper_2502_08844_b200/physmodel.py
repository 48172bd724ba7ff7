"""Model of the articulated contact physics step.

``PhysModel`` mirrors the C struct ``dk_phys_model`` (include/deskrl_b200.h)
field for field; ``go1_model()`` is the Go1-shaped quadruped the bench and
tests run.  The reference has no such model (SPEC.md:8 puts MuJoCo/MJX and the
contact-rich environments out of scope; PAPER.md:580 fixes feet-only
collision for the joystick tasks), so the numbers below are Go1-like values
in the spirit of MuJoCo Menagerie's unitree_go1 and MuJoCo Playground's Go1
joystick (timestep 0.004 s, control every 0.02 s, Kp 35, Kd 0.5) -- a
stand-in with the right shape (18 DoF, 4 feet), not a pinned asset.

This module is plain data (no CUDA): tests use it on CPU to build the model
for the oracle, and ``physics.DevicePhysics`` hands the same struct to the
sm_100a library.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

NQ, NV, NU, NBODY, MAXCON, NSENSOR = 19, 18, 12, 13, 16, 46
LIMBS = ("FR", "FL", "RR", "RL")
# geom ids (include/deskrl_b200.h): 0 floor, 1 trunk box, 2+2l thigh capsule, 3+2l foot
GEOM_FLOOR, GEOM_TRUNK = 0, 1


def geom_thigh(limb: int) -> int:
    return 2 + 2 * limb


def geom_foot(limb: int) -> int:
    return 3 + 2 * limb


_A3 = ctypes.c_double * 3
_L3x3 = ((ctypes.c_double * 3) * 3) * 4
_L3 = (ctypes.c_double * 3) * 4
_L3x2 = ((ctypes.c_double * 2) * 3) * 4


class PhysModelC(ctypes.Structure):
    _fields_ = [
        ("timestep", ctypes.c_double), ("gravity", _A3), ("friction", ctypes.c_double),
        ("solref", ctypes.c_double * 2), ("solimp", ctypes.c_double),
        ("base_mass", ctypes.c_double), ("base_ipos", _A3), ("base_inertia", _A3),
        ("base_box", _A3),
        ("body_pos", _L3x3), ("jnt_axis", _L3x3), ("body_mass", _L3), ("body_ipos", _L3x3),
        ("body_inertia", _L3x3), ("jnt_range", _L3x2), ("dof_damping", _L3),
        ("dof_armature", _L3), ("torque_limit", _L3), ("kp", ctypes.c_double),
        ("kd", ctypes.c_double), ("foot_pos", _L3), ("foot_radius", ctypes.c_double),
        ("thigh_radius", ctypes.c_double),
        ("iterations", ctypes.c_int32), ("ls_iterations", ctypes.c_int32),
        ("collide_box", ctypes.c_int32), ("collide_thigh", ctypes.c_int32),
    ]


def _limbs(fn):
    """[4][...] array from a function of (front sign fx, side sign sy)."""
    return np.array([fn(fx, sy) for fx, sy in ((1, -1), (1, 1), (-1, -1), (-1, 1))],
                    dtype=np.float64)


@dataclass
class PhysModel:
    timestep: float = 0.004
    gravity: tuple = (0.0, 0.0, -9.81)
    friction: float = 0.6
    solref: tuple = (0.02, 1.0)
    solimp: float = 0.9
    base_mass: float = 5.204
    base_ipos: tuple = (0.0223, 0.002, -0.0005)
    base_inertia: tuple = (0.0168128557, 0.063009565, 0.0716547275)
    base_box: tuple = (0.1881, 0.04675, 0.057)
    body_pos: np.ndarray = field(default_factory=lambda: _limbs(lambda fx, sy: [
        [0.1881 * fx, 0.04675 * sy, 0.0], [0.0, 0.08 * sy, 0.0], [0.0, 0.0, -0.213]]))
    jnt_axis: np.ndarray = field(default_factory=lambda: _limbs(lambda fx, sy: [
        [1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 1.0, 0.0]]))
    body_mass: np.ndarray = field(default_factory=lambda: _limbs(lambda fx, sy: [
        0.680, 1.009, 0.195862]))
    body_ipos: np.ndarray = field(default_factory=lambda: _limbs(lambda fx, sy: [
        [-0.005657 * fx, 0.008752 * sy, -0.000102], [-0.003342, -0.018054 * sy, -0.033451],
        [0.00429862, 0.000976676 * sy, -0.146197]]))
    body_inertia: np.ndarray = field(default_factory=lambda: _limbs(lambda fx, sy: [
        [0.000334008, 0.000619101, 0.00040057], [0.00443176, 0.00448537, 0.000740309],
        [0.0011454, 0.0011588, 0.0000266]]))
    jnt_range: np.ndarray = field(default_factory=lambda: _limbs(lambda fx, sy: [
        [-0.863, 0.863], [-0.686, 4.501], [-2.818, -0.888]]))
    dof_damping: np.ndarray = field(default_factory=lambda: _limbs(lambda fx, sy: [0.1] * 3))
    dof_armature: np.ndarray = field(default_factory=lambda: _limbs(lambda fx, sy: [0.005] * 3))
    torque_limit: np.ndarray = field(default_factory=lambda: _limbs(lambda fx, sy: [
        23.7, 23.7, 35.55]))
    kp: float = 35.0
    kd: float = 0.5
    foot_pos: np.ndarray = field(default_factory=lambda: _limbs(lambda fx, sy: [0.0, 0.0, -0.213]))
    foot_radius: float = 0.023
    thigh_radius: float = 0.0245
    iterations: int = 4
    ls_iterations: int = 8
    collide_box: int = 0    # feet-only collision unless enabled
    collide_thigh: int = 0

    def to_c(self) -> PhysModelC:
        c = PhysModelC()
        for name, ctype in PhysModelC._fields_:
            v = getattr(self, name)
            if isinstance(ctype, type) and issubclass(ctype, ctypes.Array):
                arr = np.asarray(v, dtype=np.float64)
                ctypes.memmove(ctypes.addressof(getattr(c, name)), arr.ctypes.data, arr.nbytes)
            else:
                setattr(c, name, v)
        return c

    @classmethod
    def from_c(cls, c: PhysModelC) -> "PhysModel":
        kw = {}
        for name, ctype in PhysModelC._fields_:
            v = getattr(c, name)
            if isinstance(ctype, type) and issubclass(ctype, ctypes.Array):
                arr = np.ctypeslib.as_array(v).astype(np.float64).copy()
                kw[name] = tuple(arr.tolist()) if arr.ndim == 1 else arr
            else:
                kw[name] = v
        return cls(**kw)

    def validate(self):
        """The C library's create-time checks, restated (ConfigError names)."""
        from .envkit import ConfigError

        if not self.timestep > 0:
            raise ConfigError("timestep must be > 0")
        if not (0.0 < self.solimp < 1.0):
            raise ConfigError("solimp must be in (0, 1)")
        if not (self.solref[0] > 0 and self.solref[1] > 0):
            raise ConfigError("solref must be positive")
        if self.iterations < 1 or self.ls_iterations < 1:
            raise ConfigError("iterations and ls_iterations must be >= 1")
        return self

    @property
    def total_mass(self) -> float:
        return float(self.base_mass + np.sum(self.body_mass))


def go1_model(**overrides) -> PhysModel:
    """The Go1-shaped quadruped (feet-only collision by default)."""
    return PhysModel(**overrides)


HOME_JOINTS = (0.0, 0.9, -1.8)
HOME_HEIGHT = 0.278


def home_qpos(n: int = 1) -> np.ndarray:
    """Playground's Go1 'home' keyframe: trunk 0.278 m up, legs (0, 0.9, -1.8)."""
    q = np.zeros((n, NQ))
    q[:, 2] = HOME_HEIGHT
    q[:, 3] = 1.0
    q[:, 7:] = np.tile(HOME_JOINTS, 4)
    return q


__all__ = ["GEOM_FLOOR", "GEOM_TRUNK", "HOME_JOINTS", "LIMBS", "MAXCON", "NBODY", "NQ",
           "NSENSOR", "NU", "NV", "PhysModel", "PhysModelC", "geom_foot", "geom_thigh",
           "go1_model", "home_qpos"]
