"""GPU parity of the articulated contact physics step (SURVEY.md §8a G1-G4,
csrc/physics.cuh) against the independent fp64 oracle (oracle/physics.c,
pinned by physics known-answer tests in tests/test_oracle_physics.py).

PARITY UNPINNED: the reference has no contact physics.

Tolerances (DESIGN.md §4 "Go1 physics"):
  * contact counts and (floor, geom) pairs: bit-exact in float64 at every step
    of a 100-step horizon; in float32 from identical states, except pairs
    whose distance is within 1e-5 m of the activation threshold;
  * float64: mass matrix / bias / kinematics 1e-11 relative (floor 1e-3); one
    step 1e-9; 100 steps 1e-7 (floor 1e-3): the oracle's dense Cholesky and
    the kernel's arrow factorisation round differently, nothing else differs;
  * float32, one step from identical float32 states: per world, the inf-norm
    error of qpos / qvel relative to max(inf-norm of the reference, 1) within
    1e-5 (qacc 1e-4: accelerations of ~1e3 rad/s^2 on the light leg links);
  * float32, 100 steps: chaotic divergence -- contact switching amplifies
    rounding -- is compared with the float64 oracle's own divergence under
    float32 state rounding (the "envelope"): the fraction of worlds beyond 1e-3
    may not exceed the envelope's by more than 2x + 0.5%, and the median world
    stays within 1e-4.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2502_08844_b200 import physics

    return physics


@pytest.fixture(scope="module")
def op():
    from oracle import physics

    return physics


def _rel(a, b, floor):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float((np.abs(a - b) / np.maximum(np.abs(b), floor)).max()) if a.size else 0.0


def _nw(a, b):
    """per-world inf-norm error relative to max(inf-norm of b, 1)"""
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.abs(a - b).reshape(len(a), -1).max(1) / np.maximum(
        np.abs(b).reshape(len(b), -1).max(1), 1.0)


def _models():
    from paper_2502_08844_b200 import physmodel as pm

    return {"feet": pm.go1_model(), "full": pm.go1_model(collide_box=1, collide_thigh=1)}


def _states(op, n, seed, cfg):
    qpos, qvel, ctrl = op.random_states(n, seed=seed)
    if cfg == "full":  # some trunks low enough for box corners and thighs to touch
        qpos[: n // 4, 2] = np.random.default_rng(seed + 1).uniform(0.02, 0.12, n // 4)
    return qpos, qvel, ctrl


def _r32(x):
    return np.asarray(x).astype(np.float32).astype(np.float64)


@pytest.mark.parametrize("cfg", ["feet", "full"])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_inspect_mass_matrix_bias_kinematics(P, op, cfg, dtype):
    """G1: forward kinematics, the CRB mass matrix and the RNE bias against the
    oracle's body-Jacobian mass matrix and generic-tree RNE."""
    model = _models()[cfg]
    n = 4096
    qpos, qvel, _ = _states(op, n, 3, cfg)
    if dtype == "float32":
        qpos, qvel = _r32(qpos), _r32(qvel)
    ref = op.inspect(model.to_c(), qpos, qvel)
    sim = P.DevicePhysics(model, n, dtype=dtype)
    t = lambda x: torch.as_tensor(x, device="cuda", dtype=sim.dtype)  # noqa: E731
    sim.set_state(t(qpos), t(qvel))
    got = {k: v.double().cpu().numpy() for k, v in sim.inspect().items()}
    if dtype == "float64":
        for k in ("M", "qfrc_bias", "xpos", "xipos"):
            assert _rel(got[k], ref[k], 1e-3) < 1e-11, k
    else:
        for k in ("xpos", "xipos"):
            assert np.abs(got[k] - ref[k]).max() < 1e-6, k
        assert _nw(got["M"], ref["M"]).max() < 1e-5
        assert _nw(got["qfrc_bias"], ref["qfrc_bias"]).max() < 1e-5
    sim.close()


@pytest.mark.parametrize("cfg", ["feet", "full"])
def test_step_f64_bitexact_contacts_and_horizon(P, op, cfg):
    """G2-G4 float64: one step and a 100-step horizon; contact counts and pairs
    bit-exact at every step, solver iteration counts equal."""
    model = _models()[cfg]
    n = 2048
    qpos, qvel, ctrl = _states(op, n, 5, cfg)
    sim = P.DevicePhysics(model, n, dtype="float64")
    t = lambda x: torch.as_tensor(x, device="cuda", dtype=torch.float64)  # noqa: E731
    sim.set_state(t(qpos), t(qvel))
    c = t(ctrl)
    qp_r, qv_r = qpos.copy(), qvel.copy()
    for s in range(100):
        out = sim.step(c, 1)
        ref = op.step(model.to_c(), qp_r, qv_r, ctrl, 1)
        qp_r, qv_r = ref["qpos"], ref["qvel"]
        o = {k: v.cpu().numpy() for k, v in out.items()}
        np.testing.assert_array_equal(o["ncon"], ref["ncon"])
        np.testing.assert_array_equal(o["contact_geom"], ref["contact_geom"])
        if s == 0:
            assert ref["ncon"].sum() > 0
            np.testing.assert_array_equal(o["solver_iter"], ref["solver_iter"])
            for k in ("qacc", "qfrc_bias", "qfrc_constraint", "contact_force", "sensordata"):
                assert _rel(o[k], ref[k], 1e-3) < 1e-9, k
            np.testing.assert_array_equal(o["act_force"], ref["act_force"])
            assert _rel(o["contact_dist"], ref["contact_dist"], 1e-3) < 1e-12
            assert _rel(o["contact_pos"], ref["contact_pos"], 1e-3) < 1e-12
            qp, qv = (x.cpu().numpy() for x in sim.state())
            assert _rel(qp, qp_r, 1e-3) < 1e-9 and _rel(qv, qv_r, 1e-3) < 1e-9
    sim.check()
    qp, qv = (x.cpu().numpy() for x in sim.state())
    assert _rel(qp, qp_r, 1e-3) < 1e-7
    assert _rel(qv, qv_r, 1e-3) < 1e-7
    sim.close()


@pytest.mark.parametrize("cfg", ["feet", "full"])
def test_step_f32_one_step(P, op, cfg):
    model = _models()[cfg]
    n = 8192
    qpos, qvel, ctrl = (_r32(x) for x in _states(op, n, 7, cfg))
    ref = op.step(model.to_c(), qpos, qvel, ctrl, 1)
    sim = P.DevicePhysics(model, n, dtype="float32")
    t = lambda x: torch.as_tensor(x, device="cuda", dtype=torch.float32)  # noqa: E731
    sim.set_state(t(qpos), t(qvel))
    out = sim.step(t(ctrl), 1)
    sim.check()
    o = {k: v.cpu().numpy() for k, v in out.items()}
    qp, qv = (x.double().cpu().numpy() for x in sim.state())
    # contacts: equal unless the reference distance is within 1e-5 m of zero
    near = (np.abs(ref["contact_dist"]) < 1e-5).any(1)
    eq = (o["contact_geom"] == ref["contact_geom"]).all(axis=(1, 2)) & (o["ncon"] == ref["ncon"])
    assert (eq | near).all(), int((~eq & ~near).sum())
    assert eq.mean() > 0.999
    assert _nw(qp[eq], ref["qpos"][eq]).max() < 1e-5
    assert _nw(qv[eq], ref["qvel"][eq]).max() < 1e-5
    assert _nw(o["qacc"][eq], ref["qacc"][eq]).max() < 1e-4
    assert _nw(o["sensordata"][eq], ref["sensordata"][eq]).max() < 1e-5
    sim.close()


def test_step_f32_horizon_vs_rounding_envelope(P, op):
    """100 steps: the float32 kernel's divergence from the fp64 oracle against
    the oracle's own divergence when only its state is rounded to float32."""
    model = _models()["feet"]
    n = 2048
    qpos, qvel, ctrl = (_r32(x) for x in _states(op, n, 11, "feet"))
    sim = P.DevicePhysics(model, n, dtype="float32")
    t = lambda x: torch.as_tensor(x, device="cuda", dtype=torch.float32)  # noqa: E731
    sim.set_state(t(qpos), t(qvel))
    sim.step(t(ctrl), 100, diag=False)
    sim.check()
    qp, qv = (x.double().cpu().numpy() for x in sim.state())
    ref = op.step(model.to_c(), qpos, qvel, ctrl, 100)
    qe, ve = qpos.copy(), qvel.copy()
    for _ in range(100):
        e = op.step(model.to_c(), qe, ve, ctrl, 1)
        qe, ve = _r32(e["qpos"]), _r32(e["qvel"])
    for a, b, env in ((qp, ref["qpos"], qe), (qv, ref["qvel"], ve)):
        nw, nwe = _nw(a, b), _nw(env, b)
        print("gpu: p50 %.2e p99 %.2e >1e-3 %.4f | envelope: p50 %.2e p99 %.2e >1e-3 %.4f" % (
            np.median(nw), np.percentile(nw, 99), (nw > 1e-3).mean(), np.median(nwe),
            np.percentile(nwe, 99), (nwe > 1e-3).mean()))
        assert np.median(nw) < 1e-4
        assert (nw > 1e-3).mean() <= 2 * (nwe > 1e-3).mean() + 0.005


def test_free_fall_and_stance_on_device(P):
    """Physics KATs on the kernel itself: free-fall acceleration of the trunk
    at zero velocity with legs locked by the PD loop is g (no contacts), and a
    robot standing on its PD targets comes to rest carrying its weight."""
    from paper_2502_08844_b200 import physmodel as pm

    m = pm.go1_model()
    n = 64
    sim = P.DevicePhysics(m, n, dtype="float64")
    q = pm.home_qpos(n)
    q[:, 2] = 3.0
    sim.reset(q)
    out = sim.step(torch.as_tensor(q[:, 7:], device="cuda", dtype=torch.float64), 1)
    assert (out["ncon"] == 0).all()
    np.testing.assert_allclose(out["qacc"][:, :3].cpu().numpy(),
                               np.tile([0, 0, -9.81], (n, 1)), atol=1e-9)
    sim.reset()
    home = torch.as_tensor(pm.home_qpos(n)[:, 7:], device="cuda", dtype=torch.float64)
    sim.step(home, 1499, diag=False)
    out = sim.step(home, 1)
    sim.check()
    qp, qv = sim.state()
    assert qv.abs().max().item() < 1e-3
    assert (out["ncon"] == 4).all()
    fn = out["contact_force"][:, :4, 0].sum(1).cpu().numpy()
    np.testing.assert_allclose(fn, m.total_mass * 9.81, rtol=1e-3)
    sim.close()


def test_bad_state_is_reported(P):
    from paper_2502_08844_b200 import InvalidInputError

    sim = P.DevicePhysics(None, 32, dtype="float32")
    sim.reset()
    ctrl = torch.full((32, 12), float("nan"), device="cuda")
    qp = torch.as_tensor(np.full((32, 19), np.nan), device="cuda", dtype=torch.float32)
    sim.set_state(qp, None)
    sim.step(ctrl, 1)
    with pytest.raises(InvalidInputError, match="not positive definite"):
        sim.check()
    with pytest.raises(InvalidInputError):
        sim.step(torch.zeros((31, 12), device="cuda"), 1)
    sim.close()
