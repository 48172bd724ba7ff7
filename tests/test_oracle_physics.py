"""Known-answer tests pinning the fp64 physics oracle (oracle/physics.c).

The reference has no contact physics, so the oracle of SURVEY.md
§8a G1-G4 cannot be checked against golden vectors ("parity unpinned").  These
tests pin it against physics instead, each through a code path independent of
the one under test:
  * inverse dynamics (RNE with qacc) == M qacc + bias (M from body Jacobians);
  * 1/2 qvel^T M qvel == kinetic energy summed from body velocities;
  * free fall: the trunk-plus-legs centre of mass accelerates at exactly g;
  * without gravity / contacts / actuation, linear and angular momentum drift
    per step is O(h^2) (a wrong Coriolis term would make it O(h));
  * analytic foot heights at the home keyframe, contact count / geoms;
  * standing still on the PD targets: contact normal forces carry the weight;
  * a joint past its range is pushed back.
"""

import numpy as np
import pytest

from oracle import physics as op
from paper_2502_08844_b200 import physmodel as pm


@pytest.fixture(scope="module")
def model():
    return pm.go1_model()


def _no_forces(model, gravity=True):
    m = pm.go1_model(kp=0.0, kd=0.0, dof_damping=np.zeros((4, 3)),
                     gravity=model.gravity if gravity else (0.0, 0.0, 0.0))
    m.jnt_range = np.tile([[-100.0, 100.0]], (4, 3, 1))  # no limit rows
    return m


def test_model_struct_roundtrip(model):
    c = model.to_c()
    back = pm.PhysModel.from_c(c)
    assert back.timestep == model.timestep and back.iterations == model.iterations
    np.testing.assert_array_equal(back.body_pos, model.body_pos)
    np.testing.assert_array_equal(back.jnt_range, model.jnt_range)


def test_mass_matrix_spd_and_inverse_dynamics(model):
    qpos, qvel, _ = op.random_states(64, seed=1)
    ins = op.inspect(model.to_c(), qpos, qvel)
    M = ins["M"]
    np.testing.assert_allclose(M, np.swapaxes(M, 1, 2), rtol=0, atol=1e-14)
    assert (np.linalg.eigvalsh(M) > 0).all()
    # trunk translation block = total mass
    for w in range(4):
        np.testing.assert_allclose(M[w, :3, :3], model.total_mass * np.eye(3), atol=1e-12)
    qacc = np.random.default_rng(2).normal(size=(64, pm.NV))
    tau = op.inverse(model.to_c(), qpos, qvel, qacc)
    np.testing.assert_allclose(tau, np.einsum("nij,nj->ni", M, qacc) + ins["qfrc_bias"],
                               rtol=1e-11, atol=1e-11)


def test_kinetic_energy_from_body_velocities(model):
    qpos, qvel, _ = op.random_states(64, seed=3)
    M = op.inspect(model.to_c(), qpos, qvel)["M"]
    arm = np.concatenate([np.zeros(6), model.dof_armature.reshape(-1)])
    ke, _, _ = op.energy(model.to_c(), qpos, qvel)
    ke_m = 0.5 * np.einsum("ni,nij,nj->n", qvel, M - np.diag(arm), qvel)
    np.testing.assert_allclose(ke_m, ke, rtol=1e-12)


def test_free_fall_com_accelerates_at_g(model):
    m = _no_forces(model)
    qpos, _, ctrl = op.random_states(32, seed=4, height=5.0)  # far above the floor
    qvel = np.zeros((32, pm.NV))
    out = op.step(m.to_c(), qpos, qvel, ctrl)
    assert (out["ncon"] == 0).all()
    # momentum is linear in the velocity: P(q, qacc) = d/dt P at qvel = 0
    _, _, mom = op.energy(m.to_c(), qpos, out["qacc"])
    np.testing.assert_allclose(mom[:, :3], np.tile(np.array(m.gravity) * m.total_mass, (32, 1)),
                               rtol=0, atol=1e-10)


@pytest.mark.parametrize("what", ["linear", "angular"])
def test_momentum_drift_is_second_order(model, what):
    qpos, qvel, ctrl = op.random_states(16, seed=5, height=5.0)
    drift = []
    for h in (1e-3, 5e-4):
        m = _no_forces(model, gravity=False)
        m.timestep = h
        out = op.step(m.to_c(), qpos, qvel, ctrl)
        _, _, p0 = op.energy(m.to_c(), qpos, qvel)
        _, _, p1 = op.energy(m.to_c(), out["qpos"], out["qvel"])
        sl = slice(0, 3) if what == "linear" else slice(3, 6)
        drift.append(np.abs(p1[:, sl] - p0[:, sl]).max())
    assert drift[0] < 1e-4
    ratio = drift[0] / max(drift[1], 1e-300)
    assert 3.0 < ratio < 5.0, (drift, ratio)  # O(h^2): halving h quarters the drift


def test_energy_drift_is_second_order(model):
    qpos, qvel, ctrl = op.random_states(16, seed=6, height=5.0)
    drift = []
    for h in (1e-3, 5e-4):
        m = _no_forces(model)
        m.timestep = h
        out = op.step(m.to_c(), qpos, qvel, ctrl)
        k0, u0, _ = op.energy(m.to_c(), qpos, qvel)
        k1, u1, _ = op.energy(m.to_c(), out["qpos"], out["qvel"])
        drift.append(np.abs((k1 + u1) - (k0 + u0)).max())
    ratio = drift[0] / drift[1]
    assert 3.0 < ratio < 5.0, (drift, ratio)


def test_home_pose_feet_heights_and_contacts(model):
    qpos = pm.home_qpos(1)
    out = op.step(model.to_c(), qpos, np.zeros((1, pm.NV)), qpos[:, 7:])
    foot_z = pm.HOME_HEIGHT - 2 * 0.213 * np.cos(0.9)
    assert out["ncon"][0] == 4
    assert out["contact_geom"][0, :4, 1].tolist() == [pm.geom_foot(l) for l in range(4)]
    assert (out["contact_geom"][0, :4, 0] == 0).all()
    np.testing.assert_allclose(out["contact_dist"][0, :4], foot_z - model.foot_radius, atol=1e-15)
    # trunk box and thigh capsules when enabled: thighs are above ground, box is not
    m2 = pm.go1_model(collide_box=1, collide_thigh=1)
    out2 = op.step(m2.to_c(), qpos, np.zeros((1, pm.NV)), qpos[:, 7:])
    assert out2["ncon"][0] == 4
    low = pm.home_qpos(1)
    low[0, 2] = 0.05  # trunk nearly on the floor: box corners and knees touch
    out3 = op.step(m2.to_c(), low, np.zeros((1, pm.NV)), low[:, 7:])
    geoms = out3["contact_geom"][0, :out3["ncon"][0], 1].tolist()
    assert geoms == sorted(geoms) and pm.GEOM_TRUNK in geoms
    assert any(g in geoms for g in [pm.geom_thigh(l) for l in range(4)])


def test_standing_carries_the_weight(model):
    qpos = pm.home_qpos(1)
    qvel = np.zeros((1, pm.NV))
    ctrl = qpos[:, 7:].copy()
    out = op.step(model.to_c(), qpos, qvel, ctrl, num_steps=1500)  # 6 s: settled
    assert np.abs(out["qvel"]).max() < 1e-3
    nc = out["ncon"][0]
    assert nc == 4
    fn = out["contact_force"][0, :nc, 0].sum()
    np.testing.assert_allclose(fn, model.total_mass * 9.81, rtol=1e-3)
    assert 0.15 < out["qpos"][0, 2] < 0.30
    assert out["solver_iter"][0] >= 1


def test_joint_limit_pushes_back(model):
    qpos = pm.home_qpos(1)
    qpos[0, 2] = 5.0
    qpos[0, 7 + 2] = model.jnt_range[0, 2, 1] + 0.05  # FR knee past its upper limit
    m = pm.go1_model(kp=0.0, kd=0.0)
    out = op.step(m.to_c(), qpos, np.zeros((1, pm.NV)), qpos[:, 7:])
    assert out["qfrc_constraint"][0, 6 + 2] < 0  # pushes towards the range


def test_library_default_model_equals_python_model():
    """dk_phys_default_model (C ABI, no GPU needed) == physmodel.go1_model()."""
    import ctypes

    from paper_2502_08844_b200 import physics

    c = physics.default_model_c()
    py = pm.go1_model().to_c()
    assert bytes(c) == bytes(py)
    assert ctypes.sizeof(c) == 2016  # sizeof(dk_phys_model) in C


def test_library_default_go1_config_equals_python_config():
    import ctypes

    from paper_2502_08844_b200 import _native as nat
    from paper_2502_08844_b200.go1env import Go1Config, Go1ConfigC

    c = Go1ConfigC()
    assert nat.lib().dk_go1_default_config(ctypes.byref(c)) == 0
    assert bytes(c) == bytes(Go1Config().to_c())
