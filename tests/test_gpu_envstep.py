"""GPU parity of the B200 env step against the reference (golden fixtures) and
the C oracle, through the C ABI (libdeskrl_b200.so).

Tolerances (BASELINE.md "Parity"):
  * flags, step / episode counters, truncation and autoreset placement: exact;
  * float64 build: reset states bit-exact; trajectories within 1e-9 relative
    (the only differences are CUDA vs glibc sin/cos/exp ulps, amplified by the
    chaotic dynamics over the horizon);
  * float32 build: 1 step within 1e-5 relative, <=100 steps within 1e-3
    relative, against max(|ref|, floor_c) with per-component
    floors derived from float32 rounding (tests/f32_envelope.py: at least
    1e-3, more only where a correctly rounded float32 restatement already
    deviates: K=4 times the deviation float32 state storage alone causes in
    the float64 oracle).  Chaotic divergence beyond ~200 steps is checked
    statistically instead.  Measured tables: profiles/r02_parity_vs_oracle.json,
    profiles/r02_f32_ab.json (product vs correctly rounded build).
"""

import numpy as np
import pytest

from tests import f32_envelope as fe

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

TASKS = ["pendulum-swingup", "cartpole-balance", "acrobot-swingup", "reacher-easy"]


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2502_08844_b200 as p

    return p


def _close(got, want, rtol, floor):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    err = np.abs(got - want) / np.maximum(np.abs(want), floor)
    return float(err.max()) if err.size else 0.0


def _traj_names(golden):
    return sorted({k.split("/")[1] for k in golden.files if k.startswith("traj/")})


def _make_params(pkg, kind):
    if kind == "damped":
        return pkg.DynamicsParams(link_damping=0.1, link2_mass=1.3, elbow_torque_limit=6.0)
    return None


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_golden_trajectories(golden, pkg, oracle, dtype):
    """BatchEnv (drop-in numpy API) replays the reference's own trajectories.
    float32: per-component floors from float32 rounding (tests/f32_envelope.py),
    1e-5 on the first step, 1e-3 after."""
    for name in _traj_names(golden):
        g = lambda k: golden[f"traj/{name}/{k}"]  # noqa: E731
        dt = float(g("meta_dt"))
        task, n = str(g("meta_task")), int(g("meta_n"))
        kw = dict(episode_length=int(g("meta_ep_len")), action_repeat=int(g("meta_rep")),
                  wide_init=bool(g("meta_wide")))
        params = _make_params(pkg, str(g("meta_params")))
        cfg = pkg.EnvConfig(task=task, dt=None if dt < 0 else dt, **kw)
        env = pkg.BatchEnv(cfg, n, params=params, dtype=dtype)
        acts = g("acts")
        if dtype == "float64":
            floor_k = lambda k: 1e-3  # noqa: E731
            tol_k = lambda k: 1e-9  # noqa: E731
            floor0, tol0 = 1e-3, 1e-12
            tol_r = tol_k
        else:
            o_ref, E = fe.envelope(oracle, task, n, int(g("meta_seed")), acts,
                                   mid_reset_step=int(g("mid_reset_step")),
                                   dt=None if dt < 0 else dt, params=params, **kw)
            np.testing.assert_allclose(o_ref, g("obs"), rtol=1e-12, atol=1e-12)  # oracle pinned
            floor_k = lambda k: fe.floors(E[k], fe.RTOL_1 if k == 0 else fe.RTOL_H)  # noqa: E731
            tol_k = lambda k: fe.RTOL_1 if k == 0 else fe.RTOL_H  # noqa: E731
            # reset states: the float32 rounding of the f64 draw
            floor0 = fe.floors(fe.reset_envelope(oracle, task, n, int(g("meta_seed")),
                                                 dt=None if dt < 0 else dt, params=params, **kw),
                               fe.RTOL_1)
            tol0 = fe.RTOL_1
            tol_r = lambda k: 1e-4 if k == 0 else 1e-3  # noqa: E731  (reward, info terms)
        obs0 = env.reset(seed=int(g("meta_seed")))
        assert _close(obs0["state"], g("obs0"), 0, floor0) < tol0
        for k in range(acts.shape[0]):
            fl, tol = floor_k(k), tol_k(k)
            if k == int(g("mid_reset_step")):
                o = env.reset()
                assert _close(o["state"], g("obs_mid_reset"), 0, floor0) < max(tol0, 1e-12)
            obs, rew, done, trunc, infos = env.step(acts[k])
            assert obs["state"].dtype == np.float64 and obs["state"].shape == g("obs")[k].shape
            np.testing.assert_array_equal(obs["state"], obs["privileged_state"])
            assert _close(obs["state"], g("obs")[k], 0, fl) < tol, (name, k)
            assert _close(rew, g("rew")[k], 0, 1e-3) < tol_r(k), (name, k)
            np.testing.assert_array_equal(done, g("done")[k])
            np.testing.assert_array_equal(trunc, g("trunc")[k])
            mask = np.array(["terminal_observation" in inf for inf in infos])
            np.testing.assert_array_equal(mask, g("term_mask")[k])
            for i in np.nonzero(mask)[0]:
                t = infos[i]["terminal_observation"]
                assert _close(t["state"], g("term_obs")[k][i], 0, fl) < tol
            info = np.array([[v for kk, v in inf.items() if kk != "terminal_observation"]
                             for inf in infos])
            assert _close(info, g("info")[k], 0, 1e-3) < tol_r(k)
        s, t, steps, ep, nr = env._h.get_state()
        np.testing.assert_array_equal(steps, g("final_steps"))
        np.testing.assert_array_equal(ep, g("final_episode"))
        if dtype == "float64":
            assert _close(s, g("final_state"), 0, 1e-3) < 1e-9
        env.close()


@pytest.mark.parametrize("task", TASKS)
def test_reset_states_match_philox_oracle(pkg, oracle, task):
    n = 4096
    env = pkg.DeviceBatchEnv(pkg.EnvConfig(task=task, wide_init=task == "pendulum-swingup"), n,
                             dtype="float64", env_index_offset=12345)
    env.reset(seed=987654321)
    s, t, steps, ep, nr = env.state()
    ref = oracle.OracleBatchEnv(task, n, wide_init=task == "pendulum-swingup", env_offset=12345)
    ref.reset(seed=987654321)
    np.testing.assert_array_equal(s, ref.state)  # Philox + uniform: bit-exact
    if task == "reacher-easy":  # target = radius * (cos, sin): CUDA vs glibc trig ulp
        np.testing.assert_allclose(t, ref.target, rtol=0, atol=4e-16)
    assert (steps == 0).all() and (ep == 0).all() and not nr.any()
    # float32: exactly the float64 draw rounded to nearest
    env32 = pkg.DeviceBatchEnv(pkg.EnvConfig(task=task, wide_init=task == "pendulum-swingup"), n,
                               dtype="float32", env_index_offset=12345)
    env32.reset(seed=987654321)
    s32, *_ = env32.state()
    np.testing.assert_array_equal(s32, ref.state.astype(np.float32).astype(np.float64))


def _oracle_rollout(oracle, task, n, K, seed, acts, **kw):
    ref = oracle.OracleBatchEnv(task, n, **kw)
    ref.reset(seed=seed)
    return ref, ref.rollout(acts)


@pytest.mark.parametrize("task", TASKS)
def test_rollout_vs_oracle_f64(pkg, oracle, task):
    n, K, seed = 8192, 100, 3
    rng = np.random.default_rng(5)
    acts = rng.uniform(-1.2, 1.2, (K, n, 2 if task == "reacher-easy" else 1))
    ref, (obs, rew, done, trunc, term, mask, info) = _oracle_rollout(
        oracle, task, n, K, seed, acts, episode_length=37, action_repeat=2)
    env = pkg.DeviceBatchEnv(pkg.EnvConfig(task=task, episode_length=37, action_repeat=2), n,
                             dtype="float64")
    env.reset(seed=seed)
    out = env.rollout(torch.as_tensor(acts, device="cuda"), with_info=True)
    env.check()
    np.testing.assert_array_equal(out["trunc"].cpu().numpy(), trunc)
    np.testing.assert_array_equal(out["done"].cpu().numpy(), done)
    np.testing.assert_array_equal(out["terminal_mask"].cpu().numpy(), mask)
    assert _close(out["obs"].cpu().numpy(), obs, 0, 1e-3) < 1e-9
    assert _close(out["reward"].cpu().numpy(), rew, 0, 1e-3) < 1e-9
    assert _close(out["info"].cpu().numpy(), info, 0, 1e-3) < 1e-9
    m = mask
    assert _close(out["terminal_obs"].cpu().numpy()[m], term[m], 0, 1e-3) < 1e-9
    s, t, steps, ep, nr = env.state()
    np.testing.assert_array_equal(steps, ref.steps)
    np.testing.assert_array_equal(ep, ref.episode)


@pytest.mark.parametrize("task", TASKS + ["pendulum-swingup/wide"])
def test_rollout_vs_oracle_f32(pkg, oracle, task):
    """8192 worlds x 100 steps: 1e-5 after 1 step, 1e-3 over 100 steps, with
    the rounding-derived floors of tests/f32_envelope.py (printed)."""
    wide = task.endswith("/wide")
    task = task.split("/")[0]
    n, K, seed = 8192, 100, 11
    rng = np.random.default_rng(6)
    # the kernel's inputs are float32: the oracle runs on the same values
    acts = fe.r32(rng.uniform(-1, 1, (K, n, 2 if task == "reacher-easy" else 1)))
    obs_ref, E = fe.envelope(oracle, task, n, seed, acts, episode_length=1000, wide_init=wide)
    ref, (obs, rew, done, trunc, term, mask, info) = _oracle_rollout(
        oracle, task, n, K, seed, acts, episode_length=1000, wide_init=wide)
    np.testing.assert_array_equal(obs, obs_ref)
    env = pkg.DeviceBatchEnv(pkg.EnvConfig(task=task, wide_init=wide), n, dtype="float32")
    env.reset(seed=seed)
    out = env.rollout(torch.as_tensor(acts, device="cuda", dtype=torch.float32), with_info=True)
    env.check()
    got = out["obs"].cpu().numpy()
    f1, f100 = fe.floors(E[0], fe.RTOL_1), fe.floors(E[-1], fe.RTOL_H)
    print(task, "wide" if wide else "", "floors@1", f1, "floors@100", f100)
    e1 = fe.rel_err(got[0], obs[0], f1)
    e100 = fe.rel_err(got, obs, f100)
    assert e1 < fe.RTOL_1, (e1, f1)
    assert e100 < fe.RTOL_H, (e100, f100)
    # reward: a product / exp of the observation's state, scale 1; floor 1e-3
    assert fe.rel_err(out["reward"].cpu().numpy()[0], rew[0], 1e-3) < 1e-4
    assert fe.rel_err(out["reward"].cpu().numpy(), rew, 1e-3) < 1e-2
    np.testing.assert_array_equal(out["trunc"].cpu().numpy(), trunc)


def test_full_episode_statistics_f32(pkg, oracle):
    """1000 steps (one full episode + autoreset) at 8192 worlds, float32:
    counters exact, trajectories compared statistically after chaos sets in."""
    n, K = 8192, 1001
    acts = np.random.default_rng(0).uniform(-1, 1, (K, n, 1))
    ref, (obs, rew, done, trunc, term, mask, info) = _oracle_rollout(
        oracle, "cartpole-balance", n, K, 0, acts)
    env = pkg.DeviceBatchEnv(pkg.EnvConfig(), n, dtype="float32")
    env.reset(seed=0)
    out = env.rollout(torch.as_tensor(acts, device="cuda", dtype=torch.float32))
    env.check()
    tr = out["trunc"].cpu().numpy()
    np.testing.assert_array_equal(tr, trunc)
    assert tr[999].all() and tr.sum() == n
    # reset obs after the autoreset is a fresh Philox draw: matches again
    got = out["obs"].cpu().numpy()
    assert _close(got[999], obs[999], 0, 1e-3) < 1e-5  # fresh resets: float32 rounding only
    r = out["reward"].cpu().numpy()
    assert abs(r.mean() - rew.mean()) < 2e-3 * max(1.0, abs(rew.mean()))
    s, t, steps, ep, nr = env.state()
    np.testing.assert_array_equal(steps, ref.steps)
    np.testing.assert_array_equal(ep, ref.episode)


def test_step_equals_rollout_and_sharding(pkg):
    """K single steps == one K-step rollout; two shards == one device run."""
    n, K = 1000, 25
    acts = torch.rand((K, n, 1), device="cuda", dtype=torch.float64) * 2 - 1
    cfg = pkg.EnvConfig(task="cartpole-balance", episode_length=10)
    a = pkg.DeviceBatchEnv(cfg, n, dtype="float64")
    a.reset(seed=4)
    ro = a.rollout(acts, with_info=True)
    b = pkg.DeviceBatchEnv(cfg, n, dtype="float64")
    b.reset(seed=4)
    for k in range(K):
        o = b.step(acts[k])
        assert torch.equal(o["obs"], ro["obs"][k])
        assert torch.equal(o["reward"], ro["reward"][k])
        assert torch.equal(o["trunc"], ro["trunc"][k])
        assert torch.equal(o["info"], ro["info"][k])
    shards = [pkg.DeviceBatchEnv(cfg, n // 2, dtype="float64", env_index_offset=r * (n // 2))
              for r in range(2)]
    for s in shards:
        s.reset(seed=4)
    parts = [s.rollout(acts[:, r * (n // 2):(r + 1) * (n // 2)].contiguous())
             for r, s in enumerate(shards)]
    assert torch.equal(torch.cat([p["obs"] for p in parts], 1), ro["obs"])
    assert torch.equal(torch.cat([p["reward"] for p in parts], 1), ro["reward"])


def test_errors_are_batch_atomic(pkg):
    env = pkg.BatchEnv(pkg.EnvConfig(task="cartpole-balance", episode_length=2), 64)
    with pytest.raises(pkg.UsageError, match="environment must be reset before stepping"):
        env.step(np.zeros((64, 1)))
    env.reset(seed=0)
    before = env._h.get_state()
    a = np.zeros((64, 1))
    a[17, 0] = np.nan
    with pytest.raises(pkg.InvalidInputError, match="action contains non-finite values"):
        env.step(a)
    after = env._h.get_state()
    for x, y in zip(before, after):
        np.testing.assert_array_equal(x, y)  # nothing was stepped
    with pytest.raises(pkg.InvalidInputError, match="actions batch size mismatch"):
        env.step(np.zeros((63, 1)))
    env.step(np.zeros((64, 1)), autoreset=False)
    _, _, _, tr, infos = env.step(np.zeros((64, 1)), autoreset=False)
    assert tr.all() and all("terminal_observation" not in i for i in infos)
    with pytest.raises(pkg.UsageError):
        env.step(np.zeros((64, 1)), autoreset=False)
    env.reset()
    env.step(np.zeros((64, 1)))  # usable again after reset
    # device API: the error surfaces at check(), the worlds stay untouched
    d = pkg.DeviceBatchEnv(pkg.EnvConfig(), 256, dtype="float32")
    d.reset(seed=1)
    bad = torch.zeros((8, 256, 1), device="cuda")
    bad[5, 200, 0] = float("inf")
    d.rollout(bad)
    with pytest.raises(pkg.InvalidInputError) as e:
        d.check()
    assert (e.value.step_index, e.value.env_index) == (5, 200)
    s, t, steps, ep, nr = d.state()
    assert (steps == 0).all()


def test_drop_in_surface(pkg):
    env = pkg.BatchEnv(pkg.EnvConfig(task="reacher-easy"), 8, num_workers=4)
    assert env.num_envs == 8 and env.action_dim == 2
    obs = env.reset(seed=3)
    assert set(obs) == {"state", "privileged_state"} and obs["state"].shape == (8, 10)
    assert env.envs[0].observation_shapes() == {"state": (10,), "privileged_state": (10,)}
    assert len(env.envs[3].state) == 4
    o, r, d, t, infos = env.step(np.zeros((8, 2)))
    assert r.dtype == np.float64 and d.dtype == bool and t.dtype == bool
    assert set(infos[0]) == {"distance"}
    assert env.kernel_launches > 0
    env.close()


@pytest.mark.parametrize("n", [1, 37, 1000, 4097])
@pytest.mark.parametrize("task", ["cartpole-balance", "reacher-easy"])
def test_ragged_world_counts(pkg, oracle, n, task):
    """Partial 32-world tiles and unaligned action rows (the cp.async path
    instead of TMA bulk copies) give the same results as aligned ones."""
    K = 23
    A = 2 if task == "reacher-easy" else 1
    acts = np.random.default_rng(n).uniform(-1.1, 1.1, (K, n, A))
    ref, (obs, rew, done, trunc, term, mask, info) = _oracle_rollout(
        oracle, task, n, K, 2, acts, episode_length=9)
    _, E = fe.envelope(oracle, task, n, 2, acts, episode_length=9)
    f32_floor = fe.floors(E[-1], fe.RTOL_H)
    for dtype, tol, floor in (("float64", 1e-9, 1e-3), ("float32", 1e-3, f32_floor)):
        env = pkg.DeviceBatchEnv(pkg.EnvConfig(task=task, episode_length=9), n, dtype=dtype)
        env.reset(seed=2)
        out = env.rollout(torch.as_tensor(acts, device="cuda", dtype=env.dtype), with_info=True)
        env.check()
        assert _close(out["obs"].double().cpu().numpy(), obs, 0, floor) < tol
        assert _close(out["reward"].double().cpu().numpy(), rew, 0, 1e-3) < tol
        assert _close(out["info"].double().cpu().numpy(), info, 0, 1e-3) < tol
        np.testing.assert_array_equal(out["trunc"].cpu().numpy(), trunc)
        np.testing.assert_array_equal(out["terminal_mask"].cpu().numpy(), mask)
        m = mask
        assert _close(out["terminal_obs"].double().cpu().numpy()[m], term[m], 0, floor) < tol
        # an unaligned view of the actions (offset by one element) as well
        big = torch.zeros(K * n * A + 1, device="cuda", dtype=env.dtype)
        view = big[1:].view(K, n, A)
        view.copy_(torch.as_tensor(acts, device="cuda", dtype=env.dtype))
        env.reset(seed=2)
        out2 = env.rollout(view, with_info=True)
        env.check()
        assert torch.equal(out2["obs"], out["obs"]) and torch.equal(out2["reward"], out["reward"])


def test_single_environment_matches_batch_world(pkg, golden):
    """make_env / Environment (envkit.py:469-588) == world i of a BatchEnv."""
    cfg = pkg.EnvConfig(task="acrobot-swingup", episode_length=5)
    batch = pkg.BatchEnv(cfg, 8)
    batch.reset(seed=3)
    env = pkg.Environment(cfg, env_index=6)
    o = env.reset(seed=3)
    assert o["state"].shape == (6,)
    acts = np.random.default_rng(1).uniform(-1, 1, (5, 8, 1))
    for k in range(5):
        bo, br, bd, bt, binfo = batch.step(acts[k], autoreset=False)
        res = env.step(acts[k, 6])
        np.testing.assert_array_equal(res.observation["state"], bo["state"][6])
        assert res.reward == br[6] and res.truncated == bt[6] and not res.done
        assert res.info == binfo[6]
    with pytest.raises(pkg.UsageError):
        env.step([0.0])
    e2 = pkg.make_env("pendulum-swingup")
    e2.reset()
    assert e2.step([0.1]).observation["state"].shape == (3,)


@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_rollout_host_matches_device_rollout(pkg, dtype):
    """dk_env_rollout_host (pinned/pageable host buffers, chunked + pipelined,
    done / terminal_mask derived on the host) == the device rollout."""
    n, K, chunk = 1000, 2500, 700
    cfg = pkg.EnvConfig(task="reacher-easy", episode_length=300)
    a = pkg.DeviceBatchEnv(cfg, n, dtype=dtype)
    b = pkg.DeviceBatchEnv(cfg, n, dtype=dtype)
    a.reset(seed=1)
    b.reset(seed=1)
    npdt = np.float64 if dtype == "float64" else np.float32
    acts = np.random.default_rng(2).uniform(-1, 1, (K, n, 2)).astype(npdt)
    ref = a.rollout(torch.as_tensor(acts, device="cuda"), with_info=True)
    a.check()
    O, I = 10, 1
    obs = np.zeros((K, n, O), npdt)
    rew = np.zeros((K, n), npdt)
    done = np.ones((K, n), np.uint8)
    trunc = np.zeros((K, n), np.uint8)
    term = np.zeros((K, n, O), npdt)
    mask = np.zeros((K, n), np.uint8)
    info = np.zeros((K, n, I), npdt)
    rc = b._h._lib.dk_env_rollout_host(b._h.h, K, chunk, acts.ctypes.data, obs.ctypes.data,
                                       rew.ctypes.data, done.ctypes.data, trunc.ctypes.data,
                                       term.ctypes.data, mask.ctypes.data, info.ctypes.data)
    assert rc == 0
    np.testing.assert_array_equal(obs, ref["obs"].cpu().numpy())
    np.testing.assert_array_equal(rew, ref["reward"].cpu().numpy())
    np.testing.assert_array_equal(done, ref["done"].cpu().numpy())
    np.testing.assert_array_equal(trunc, ref["trunc"].cpu().numpy())
    np.testing.assert_array_equal(mask, ref["terminal_mask"].cpu().numpy())
    np.testing.assert_array_equal(info, ref["info"].cpu().numpy())
    m = mask.astype(bool)
    assert m.sum() == 8 * n
    np.testing.assert_array_equal(term[m], ref["terminal_obs"].cpu().numpy()[m])
