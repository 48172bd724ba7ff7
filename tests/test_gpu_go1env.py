"""GPU parity of the fused Go1 joystick env step (csrc/go1env.cuh: physics
substeps + reward + observation + termination + auto-reset in one kernel)
against oracle/go1env.py, which composes the independent physics oracle
(oracle/physics.c), the reference-pinned tail oracle (oracle/locomotion.c) and
a NumPy restatement of the gait bookkeeping.  UNPINNED.

float64: every flag (done, trunc, terminal mask, contacts through the
privileged observation) exact; rewards, observations and state within 1e-9
relative (floor 1e-3) over 60 control steps with terminations and
truncations.  float32: the first control steps per world within 1e-4 (times the step
count) in inf-norm relative to max(inf-norm of the reference, 1), the physics
tests' measure -- a control step is 5 physics steps whose float32
accelerations carry ~3e-6 normwise error each and spread over every component
through the coupled mass matrix.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2502_08844_b200 import go1env

    return go1env


def _rel(a, b, floor):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float((np.abs(a - b) / np.maximum(np.abs(b), floor)).max()) if a.size else 0.0


def _cfg(G, **kw):
    c = G.Go1Config(episode_length=25, term_height=0.22, seed=3)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


@pytest.mark.parametrize("geoms", ["feet", "full"])
def test_go1_env_f64_matches_oracle(G, geoms):
    """feet: the default feet-only collision; full: trunk box and thigh capsules
    collide too (the fused kernel with 19 constraint rows per lane)."""
    from oracle.go1env import OracleGo1Env
    from paper_2502_08844_b200 import physmodel as pm

    n, K = 64, 60
    cfg = _cfg(G)
    model = pm.go1_model(**({} if geoms == "feet" else dict(collide_box=1, collide_thigh=1)))
    env = G.DeviceGo1Env(n, cfg, model=model, dtype="float64", env_index_offset=100)
    ref = OracleGo1Env(model, cfg.oracle_dict(), n, env_index_offset=100)
    o = env.reset(seed=3)
    r_obs, r_priv = ref.reset(seed=3)
    assert _rel(o["state"].cpu().numpy(), r_obs, 1e-3) < 1e-12
    assert _rel(o["privileged_state"].cpu().numpy(), r_priv, 1e-3) < 1e-12
    acts = np.random.default_rng(0).uniform(-1.3, 1.3, (K, n, 12))
    out = env.rollout(torch.as_tensor(acts, device="cuda"), with_terms=True)
    env.check()
    got = {k: v.cpu().numpy() for k, v in out.items() if v is not None}
    n_done = n_trunc = 0
    for k in range(K):
        r = ref.step(acts[k])
        np.testing.assert_array_equal(got["done"][k].astype(bool), r["done"], err_msg=str(k))
        np.testing.assert_array_equal(got["trunc"][k].astype(bool), r["trunc"], err_msg=str(k))
        np.testing.assert_array_equal(got["terminal_mask"][k].astype(bool), r["terminal_mask"])
        n_done += int(r["done"].sum())
        n_trunc += int(r["trunc"].sum())
        assert _rel(got["reward"][k], r["reward"], 1e-3) < 1e-9, k
        assert _rel(got["terms"][k], r["terms"], 1e-3) < 1e-9, k
        assert _rel(got["obs"][k], r["obs"], 1e-3) < 1e-9, k
        assert _rel(got["privileged_state"][k], r["priv"], 1e-3) < 1e-9, k
        m = r["terminal_mask"]
        assert _rel(got["terminal_obs"][k][m], r["terminal_obs"][m], 1e-3) < 1e-9, k
    assert n_trunc > 0 and n_done > 0  # both auto-reset paths exercised
    s = {k: v.cpu().numpy() for k, v in env.state().items()}
    np.testing.assert_array_equal(s["steps"], ref.steps)
    np.testing.assert_array_equal(s["episode"], ref.episode)
    np.testing.assert_array_equal(s["last_contact"].astype(bool), ref.last_contact)
    for k, v in (("qpos", ref.qpos), ("qvel", ref.qvel), ("command", ref.cmd),
                 ("phase", ref.phase), ("airtime", ref.air), ("prev_action", ref.prev)):
        assert _rel(s[k], v, 1e-3) < 1e-9, k
    # domain randomisation: each world's friction / trunk mass / kp of its episode
    np.testing.assert_array_equal(env.params().cpu().numpy(), ref.params)
    assert np.ptp(ref.params[:, 0]) > 0.1  # the draws do vary across worlds
    env.close()


def test_go1_env_f64_multiwarp_ctas(G):
    """A world count whose CTAs span several warps (the step's CTA barriers are
    active) with a partial last CTA (no barriers there): 2003 worlds -> 126 CTAs
    of 16 worlds / 64 threads, the last one with 3 worlds."""
    from oracle.go1env import OracleGo1Env
    from paper_2502_08844_b200 import physmodel as pm

    n, K = 2003, 4
    cfg = _cfg(G)
    env = G.DeviceGo1Env(n, cfg, dtype="float64")
    ref = OracleGo1Env(pm.go1_model(), cfg.oracle_dict(), n)
    o = env.reset(seed=8)
    r_obs, _ = ref.reset(seed=8)
    assert _rel(o["state"].cpu().numpy(), r_obs, 1e-3) < 1e-12
    acts = np.random.default_rng(4).uniform(-1.3, 1.3, (K, n, 12))
    out = env.rollout(torch.as_tensor(acts, device="cuda"))
    env.check()
    for k in range(K):
        r = ref.step(acts[k])
        np.testing.assert_array_equal(out["done"][k].cpu().numpy().astype(bool), r["done"])
        assert _rel(out["reward"][k].cpu().numpy(), r["reward"], 1e-3) < 1e-9, k
        assert _rel(out["obs"][k].cpu().numpy(), r["obs"], 1e-3) < 1e-9, k
    s = env.state()
    assert _rel(s["qpos"].cpu().numpy(), ref.qpos, 1e-3) < 1e-9
    assert _rel(s["qvel"].cpu().numpy(), ref.qvel, 1e-3) < 1e-9
    env.close()


def test_go1_env_f32_first_steps(G):
    from oracle.go1env import OracleGo1Env
    from paper_2502_08844_b200 import physmodel as pm

    n, K = 256, 3
    cfg = _cfg(G, obs_noise=(0.0, 0.0, 0.0, 0.0, 0.0))
    env = G.DeviceGo1Env(n, cfg, dtype="float32")
    ref = OracleGo1Env(pm.go1_model(), cfg.oracle_dict(), n)
    o = env.reset(seed=5)
    r_obs, _ = ref.reset(seed=5)
    assert _rel(o["state"].double().cpu().numpy(), r_obs, 1e-2) < 1e-5
    acts = np.random.default_rng(1).uniform(-1, 1, (K, n, 12)).astype(np.float32)
    out = env.rollout(torch.as_tensor(acts, device="cuda"))
    env.check()
    for k in range(K):
        r = ref.step(acts[k].astype(np.float64))
        np.testing.assert_array_equal(out["done"][k].cpu().numpy().astype(bool), r["done"])
        g = out["obs"][k].double().cpu().numpy()
        nw = np.abs(g - r["obs"]).max(1) / np.maximum(np.abs(r["obs"]).max(1), 1.0)
        print(k, "obs normwise max %.2e p99 %.2e" % (nw.max(), np.percentile(nw, 99)))
        assert nw.max() < 1e-4 * (k + 1), k
        rw = out["reward"][k].double().cpu().numpy()
        assert np.abs(rw - r["reward"]).max() < 1e-4 * (k + 1) * max(1.0, np.abs(r["reward"]).max())
    env.close()


def test_go1_env_errors(G):
    from paper_2502_08844_b200 import InvalidInputError, UsageError

    env = G.DeviceGo1Env(40, _cfg(G))
    with pytest.raises(UsageError):
        env.step(torch.zeros((40, 12), device="cuda"))
    env.reset(seed=0)
    a = torch.zeros((4, 40, 12), device="cuda")
    a[2, 17, 5] = float("nan")
    env.rollout(a)
    with pytest.raises(InvalidInputError, match="non-finite") as ei:
        env.check()
    assert (ei.value.step_index, ei.value.env_index) == (2, 17)
    env.rollout(torch.zeros((2, 40, 12), device="cuda"))
    env.check()  # the error was reported once
    env.close()


def test_go1_env_world_count_invariance(G):
    """A world's trajectory does not depend on how many worlds share the launch:
    the CTA size follows the world count (one CTA per SM per wave; 1 to 64
    worlds per CTA, the step's CTA barriers only in full CTAs), so the same
    worlds stepped within batches of 5, 300 and 9001 are bit-identical, float32
    and float64."""
    K = 6
    for dt in ("float32", "float64"):
        ref = None
        for n in (9001, 300, 5):
            env = G.DeviceGo1Env(n, _cfg(G, episode_length=4), dtype=dt)
            env.reset(seed=12)
            acts = torch.as_tensor(np.random.default_rng(2).uniform(-1, 1, (K, 9001, 12))[:, :n],
                                   device="cuda", dtype=env.dtype)
            out = env.rollout(acts.contiguous())
            env.check()
            got = (out["obs"].cpu().numpy(), out["reward"].cpu().numpy(),
                   env.state()["qpos"].cpu().numpy())
            env.close()
            if ref is None:
                ref = got
                continue
            np.testing.assert_array_equal(got[0], ref[0][:, :n])
            np.testing.assert_array_equal(got[1], ref[1][:, :n])
            np.testing.assert_array_equal(got[2], ref[2][:n])
