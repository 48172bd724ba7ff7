"""ctypes front-end of the fp64 physics oracle (oracle/physics.c).

TEST INFRASTRUCTURE ONLY -- the checker for the articulated contact physics
kernels, never the thing measured or shipped.  Only
tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs import it.

PARITY UNPINNED: the reference has no contact physics, so this
oracle is pinned by physical known-answer tests (tests/test_oracle_physics.py)
instead of golden vectors.
"""

from __future__ import annotations

import ctypes

import numpy as np

from .oracle import lib as _orc_lib

NQ, NV, NU, NBODY, MAXCON, NSENSOR = 19, 18, 12, 13, 16, 46

_P = ctypes.c_void_p
_bound = False


def lib():
    global _bound
    L = _orc_lib()
    if not _bound:
        L.orc_phys_step.restype = ctypes.c_int
        L.orc_phys_step.argtypes = [_P, ctypes.c_int64, ctypes.c_int64] + [_P] * 14
        L.orc_phys_inspect.restype = None
        L.orc_phys_inspect.argtypes = [_P, ctypes.c_int64] + [_P] * 6
        L.orc_phys_inverse.restype = None
        L.orc_phys_inverse.argtypes = [_P, ctypes.c_int64] + [_P] * 4
        L.orc_phys_foot_kin.restype = None
        L.orc_phys_foot_kin.argtypes = [_P, ctypes.c_int64] + [_P] * 4
        L.orc_phys_energy.restype = None
        L.orc_phys_energy.argtypes = [_P, ctypes.c_int64] + [_P] * 5
        _bound = True
    return L


def _c(a, dt=np.float64):
    return np.ascontiguousarray(a, dtype=dt)


def step(model_c, qpos, qvel, ctrl, num_steps=1):
    """Advance copies of (qpos [N,19], qvel [N,18]) num_steps steps with ctrl
    [N,12] held.  Returns a dict: qpos, qvel and the last step's diagnostics."""
    qpos, qvel, ctrl = _c(qpos).copy(), _c(qvel).copy(), _c(ctrl)
    n = qpos.shape[0]
    out = {"qacc": np.zeros((n, NV)), "qfrc_bias": np.zeros((n, NV)),
           "qfrc_constraint": np.zeros((n, NV)), "act_force": np.zeros((n, NU)),
           "ncon": np.zeros(n, np.int32), "contact_geom": np.zeros((n, MAXCON, 2), np.int32),
           "contact_dist": np.zeros((n, MAXCON)), "contact_pos": np.zeros((n, MAXCON, 3)),
           "contact_force": np.zeros((n, MAXCON, 3)), "solver_iter": np.zeros(n, np.int32),
           "sensordata": np.zeros((n, NSENSOR))}
    bad = lib().orc_phys_step(
        ctypes.byref(model_c), n, int(num_steps), qpos.ctypes.data, qvel.ctypes.data,
        ctrl.ctypes.data, *[out[k].ctypes.data for k in (
            "qacc", "qfrc_bias", "qfrc_constraint", "act_force", "ncon", "contact_geom",
            "contact_dist", "contact_pos", "contact_force", "solver_iter", "sensordata")])
    if bad:
        raise RuntimeError(f"oracle: {bad} worlds hit a non-SPD matrix")
    out["qpos"], out["qvel"] = qpos, qvel
    return out


def inspect(model_c, qpos, qvel):
    qpos, qvel = _c(qpos), _c(qvel)
    n = qpos.shape[0]
    M = np.zeros((n, NV, NV))
    bias = np.zeros((n, NV))
    xpos = np.zeros((n, NBODY, 3))
    xipos = np.zeros((n, NBODY, 3))
    lib().orc_phys_inspect(ctypes.byref(model_c), n, qpos.ctypes.data, qvel.ctypes.data,
                           M.ctypes.data, bias.ctypes.data, xpos.ctypes.data, xipos.ctypes.data)
    return {"M": M, "qfrc_bias": bias, "xpos": xpos, "xipos": xipos}


def inverse(model_c, qpos, qvel, qacc):
    qpos, qvel, qacc = _c(qpos), _c(qvel), _c(qacc)
    n = qpos.shape[0]
    qfrc = np.zeros((n, NV))
    lib().orc_phys_inverse(ctypes.byref(model_c), n, qpos.ctypes.data, qvel.ctypes.data,
                           qacc.ctypes.data, qfrc.ctypes.data)
    return qfrc


def foot_kin(model_c, qpos, qvel):
    """foot sphere centres [N,4,3] and their world velocities [N,4,3]"""
    qpos, qvel = _c(qpos), _c(qvel)
    n = qpos.shape[0]
    pos, vel = np.zeros((n, 4, 3)), np.zeros((n, 4, 3))
    lib().orc_phys_foot_kin(ctypes.byref(model_c), n, qpos.ctypes.data, qvel.ctypes.data,
                            pos.ctypes.data, vel.ctypes.data)
    return pos, vel


def energy(model_c, qpos, qvel):
    qpos, qvel = _c(qpos), _c(qvel)
    n = qpos.shape[0]
    ke, pe, mom = np.zeros(n), np.zeros(n), np.zeros((n, 6))
    lib().orc_phys_energy(ctypes.byref(model_c), n, qpos.ctypes.data, qvel.ctypes.data,
                          ke.ctypes.data, pe.ctypes.data, mom.ctypes.data)
    return ke, pe, mom


def random_states(n, seed=0, spread=1.0, height=None):
    """Random (qpos, qvel, ctrl) around the home pose: joint angles within
    their ranges, a random trunk orientation tilt, random velocities; the trunk
    height is drawn so some feet are in contact and some are not."""
    rng = np.random.default_rng(seed)
    from paper_2502_08844_b200.physmodel import HOME_JOINTS, go1_model

    m = go1_model()
    qpos = np.zeros((n, NQ))
    qpos[:, 0:2] = rng.uniform(-1, 1, (n, 2))
    qpos[:, 2] = rng.uniform(0.22, 0.34, n) if height is None else height
    ax = rng.normal(size=(n, 3))
    ax /= np.linalg.norm(ax, axis=1, keepdims=True)
    ang = rng.uniform(-0.3, 0.3, n) * spread
    qpos[:, 3] = np.cos(ang / 2)
    qpos[:, 4:7] = ax * np.sin(ang / 2)[:, None]
    home = np.tile(HOME_JOINTS, 4)
    lo = m.jnt_range[:, :, 0].reshape(-1)
    hi = m.jnt_range[:, :, 1].reshape(-1)
    qpos[:, 7:] = np.clip(home + rng.normal(0, 0.3 * spread, (n, 12)), lo - 0.05, hi + 0.05)
    qvel = rng.normal(0, 0.5 * spread, (n, NV))
    ctrl = home + rng.normal(0, 0.3 * spread, (n, 12))
    return qpos, qvel, ctrl
