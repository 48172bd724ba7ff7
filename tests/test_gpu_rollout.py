"""On-device rollout collection against the reference's own
ppo.collect_rollout (tests/golden/rollout_golden.npz: 64 cartpole worlds,
episode_length 5 so truncation bootstraps happen inside the 8-step unroll, two
phases with observation normalisers, the reference's MLP weights and noise).

Tolerance: the networks run in float32 on cuBLAS vs the reference's CPU torch
(different summation order, ~1e-7 relative per layer) and the env in float64:
everything agrees to 1e-4 relative (floor 1e-3); truncation / done flags exactly."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gold():
    from tests.conftest import GOLDEN

    return np.load(os.path.join(GOLDEN, "rollout_golden.npz"))


def _close(a, b, floor=1e-3):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), floor)))


@pytest.mark.parametrize("which", ["small", "default"])
def test_collect_rollout_matches_reference(gold, which):
    """small: the reference's MLPs with hidden (32, 32) / (48, 48) (torch on the
    GPU); default: its default sizes 4 x 128 / 5 x 256 (tests/golden/
    rollout_golden_default.npz), served by the tensor-core MLP kernel."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2502_08844_b200 as dk
    from paper_2502_08844_b200 import mlp as TC
    from paper_2502_08844_b200 import ppo as P
    from paper_2502_08844_b200 import rollout as R
    from tests.conftest import GOLDEN

    if which == "default":
        gold = np.load(os.path.join(GOLDEN, "rollout_golden_default.npz"))
    N, T = 64, 8
    ph, vh = ((32, 32), (48, 48)) if which == "small" else ((128,) * 4, (256,) * 5)
    policy = R.make_policy(5, 1, ph).cuda()
    value = R.make_value(5, vh).cuda()
    assert TC.supported(policy.trunk) == (which == "default")
    assert TC.supported(value.trunk) == (which == "default")
    policy.load_state_dict({k[7:]: torch.as_tensor(gold[k]) for k in gold.files
                            if k.startswith("policy/")})
    value.load_state_dict({k[6:]: torch.as_tensor(gold[k]) for k in gold.files
                           if k.startswith("value/")})

    class Cfg:
        unroll_length, reward_scaling, discounting = T, 10.0, 0.995
        policy_obs_key = value_obs_key = "state"

    env = dk.DeviceBatchEnv(dk.EnvConfig(task="cartpole-balance", episode_length=5), N,
                            dtype="float64")
    obs = env.reset(seed=3)
    np.testing.assert_array_equal(obs["state"].cpu().numpy(), gold["obs0"])
    pn, vn = P.DeviceRunningNormalizer(5), P.DeviceRunningNormalizer(5)
    for phase in range(2):
        g = lambda k: gold[f"p{phase}/{k}"]  # noqa: E731
        noise = torch.as_tensor(g("noise"), device="cuda")
        batch, obs, mean_r = R.collect_rollout_device(env, policy, value, Cfg, obs, pn, vn,
                                                      noise=noise)
        np.testing.assert_array_equal(batch.dones.cpu().numpy(), g("dones"))
        for f in ("policy_obs", "value_obs", "actions", "pre_tanh", "log_probs", "rewards",
                  "values", "bootstrap"):
            err = _close(getattr(batch, f).cpu().numpy(), g(f))
            assert err < 1e-4, (phase, f, err)
        assert _close(obs["state"].cpu().numpy(), g("next_obs")) < 1e-4
        assert abs(float(mean_r) - float(g("mean_reward"))) < 1e-4
        for name, nz in (("pn", pn), ("vn", vn)):
            c, m, v = nz.to_numpy()
            assert c == float(g(f"{name}_count"))
            assert _close(m, g(f"{name}_mean"), 1e-6) < 1e-4
            assert _close(v, g(f"{name}_var"), 1e-6) < 1e-4
    env.check()


def test_rollout_graph_replay():
    """RolloutGraph: a captured phase replays with the env state advancing, the
    normaliser statistics folding in T*N rows per phase, and outputs equal to an
    eager phase run with the same noise source state."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2502_08844_b200 as dk
    from paper_2502_08844_b200 import ppo as P
    from paper_2502_08844_b200 import rollout as R

    N, T = 256, 6

    class Cfg:
        unroll_length, reward_scaling, discounting = T, 10.0, 0.995
        policy_obs_key = value_obs_key = "state"

    torch.manual_seed(0)
    policy, value = R.make_policy(5, 1, (32, 32)).cuda(), R.make_value(5, (32,)).cuda()
    env = dk.DeviceBatchEnv(dk.EnvConfig(task="cartpole-balance", episode_length=4), N)
    obs = env.reset(seed=1)
    pn, vn = P.DeviceRunningNormalizer(5), P.DeviceRunningNormalizer(5)
    rg = R.RolloutGraph(env, policy, value, Cfg, obs, pn, vn)
    assert pn.count == T * N
    for k in range(3):
        batch, obs, mr = rg.run()
        assert pn.count == (k + 2) * T * N and vn.count == (k + 2) * T * N
        d = batch.dones.cpu().numpy()
        assert d.shape == (T, N) and set(np.unique(d)) <= {0.0, 1.0}
        assert d.sum() > 0  # episode_length 4 inside a 6-step phase
        for f in ("policy_obs", "actions", "log_probs", "rewards", "values", "bootstrap"):
            assert torch.isfinite(getattr(batch, f)).all(), f
    env.check()


def test_rollout_graph_first_replay_continues_eager_phase():
    """Building a RolloutGraph must not advance the env: its first replay starts
    from exactly the worlds (state, counters) and observation where the eager
    set-up phase stopped -- the same inputs as a second eager phase -- and the
    episode counters after it equal two eager phases'."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2502_08844_b200 as dk
    from paper_2502_08844_b200 import ppo as P
    from paper_2502_08844_b200 import rollout as R

    N, T = 256, 6

    class Cfg:
        unroll_length, reward_scaling, discounting = T, 10.0, 0.995
        policy_obs_key = value_obs_key = "state"

    def setup():
        torch.manual_seed(0)
        policy, value = R.make_policy(5, 1, (32, 32)).cuda(), R.make_value(5, (32,)).cuda()
        env = dk.DeviceBatchEnv(dk.EnvConfig(task="cartpole-balance", episode_length=4), N)
        obs = env.reset(seed=1)
        return env, policy, value, obs, P.DeviceRunningNormalizer(5), P.DeviceRunningNormalizer(5)

    env_a, pa, va, obs_a, pna, vna = setup()
    rg = R.RolloutGraph(env_a, pa, va, Cfg, obs_a, pna, vna)
    env_b, pb, vb, obs_b, pnb, vnb = setup()
    _, obs_b, _ = R.collect_rollout_device(env_b, pb, vb, Cfg, obs_b, pnb, vnb)
    sa, sb = env_a.state(), env_b.state()
    for x, y in zip(sa, sb):  # construction left the env exactly after phase 1
        np.testing.assert_array_equal(x, y)
    batch_a, _, _ = rg.run()
    batch_b, _, _ = R.collect_rollout_device(env_b, pb, vb, Cfg, obs_b, pnb, vnb)
    torch.testing.assert_close(batch_a.policy_obs[0], batch_b.policy_obs[0], rtol=0, atol=0)
    torch.testing.assert_close(batch_a.value_obs[0], batch_b.value_obs[0], rtol=0, atol=0)
    sa, sb = env_a.state(), env_b.state()
    np.testing.assert_array_equal(sa[2], sb[2])  # steps
    np.testing.assert_array_equal(sa[3], sb[3])  # episode
    np.testing.assert_array_equal(batch_a.dones.cpu().numpy(), batch_b.dones.cpu().numpy())
    env_a.close()
    env_b.close()


def test_rollout_nan_policy_raises():
    """ppo.policy_forward raises RuntimeError('policy produced NaN mean')
    (ppo.py:208); the device rollout checks the flag once per phase."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2502_08844_b200 as dk
    from paper_2502_08844_b200 import rollout as R

    class Cfg:
        unroll_length, reward_scaling, discounting = 3, 10.0, 0.995
        policy_obs_key = value_obs_key = "state"

    torch.manual_seed(0)
    policy, value = R.make_policy(5, 1, (32,)).cuda(), R.make_value(5, (32,)).cuda()
    with torch.no_grad():
        for prm in policy.parameters():  # NaN weights -> NaN mean
            prm.fill_(float("nan"))
    env = dk.DeviceBatchEnv(dk.EnvConfig(task="cartpole-balance"), 64)
    obs = env.reset(seed=0)
    with pytest.raises(RuntimeError, match="policy produced NaN mean"):
        R.collect_rollout_device(env, policy, value, Cfg, obs)
    env.close()


def test_pixel_policy_rollout_matches_reference():
    """collect_rollout_device with the reference's CNNPolicy on pixel_normalize'd
    cartpole pixel stacks (tests/golden/rollout_pixels_golden.npz): the policy
    inputs equal the reference's (float32 of the float64 standardisation), the
    rest agrees to the network tolerance above (cuDNN convolutions in float32,
    TF32 off as on the reference's CPU)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2502_08844_b200 as dk
    from paper_2502_08844_b200 import ppo as P
    from paper_2502_08844_b200 import rollout as R
    from tests.conftest import GOLDEN

    g = np.load(os.path.join(GOLDEN, "rollout_pixels_golden.npz"))
    N, T = 4, 6
    policy = R.make_cnn_policy(3, 64, 1, (32,)).cuda()
    value = R.make_value(5, (48, 48)).cuda()
    policy.load_state_dict({k[7:]: torch.as_tensor(g[k]) for k in g.files
                            if k.startswith("policy/")})
    value.load_state_dict({k[6:]: torch.as_tensor(g[k]) for k in g.files
                           if k.startswith("value/")})

    class Cfg:
        unroll_length, reward_scaling, discounting = T, 10.0, 0.995
        policy_obs_key, value_obs_key = "pixels", "state"

    env = dk.DeviceBatchEnv(dk.EnvConfig(task="cartpole-balance-pixels", episode_length=4,
                                         visual_randomization=True), N, dtype="float64")
    obs = env.reset(seed=6)
    np.testing.assert_array_equal(obs["state"].cpu().numpy(), g["obs0"])
    vn = P.DeviceRunningNormalizer(5)
    tf32 = torch.backends.cudnn.allow_tf32
    torch.backends.cudnn.allow_tf32 = False
    try:
        batch, obs, mean_r = R.collect_rollout_device(
            env, policy, value, Cfg, obs, None, vn,
            noise=torch.as_tensor(g["noise"], device="cuda"))
    finally:
        torch.backends.cudnn.allow_tf32 = tf32
    po = batch.policy_obs.cpu().numpy()
    assert po.shape == (T, N, 3, 64, 64) and po.dtype == np.float32
    np.testing.assert_array_equal(po[0], g["policy_obs_first"])
    np.testing.assert_array_equal(po[-1], g["policy_obs_last"])
    np.testing.assert_allclose(po.astype(np.float64).sum(axis=(3, 4)), g["policy_obs_sums"],
                               rtol=0, atol=1e-9)
    np.testing.assert_array_equal(batch.dones.cpu().numpy(), g["dones"])
    for f in ("value_obs", "actions", "pre_tanh", "log_probs", "rewards", "values", "bootstrap"):
        err = _close(getattr(batch, f).cpu().numpy(), g[f])
        assert err < 1e-4, (f, err)
    assert _close(obs["state"].cpu().numpy(), g["next_obs"]) < 1e-4
    assert abs(float(mean_r) - float(g["mean_reward"])) < 1e-4
    c, m, v = vn.to_numpy()
    assert c == float(g["vn_count"])
    assert _close(m, g["vn_mean"], 1e-6) < 1e-4 and _close(v, g["vn_var"], 1e-6) < 1e-4
    with pytest.raises(dk.ConfigError):
        R.RolloutGraph(env, policy, value, Cfg, obs, None, vn)
    env.check()


def test_evaluate_device_matches_reference():
    """rollout.evaluate_device against ppo.evaluate (tests/golden/evaluate_golden.*):
    MLP policy with a policy normaliser (full episodes, then max_steps=10 continuing
    the episode counters) and the CNN policy on pixel stacks; returns within the
    network tolerance, the step counts exactly."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import json

    import paper_2502_08844_b200 as dk
    from paper_2502_08844_b200 import ppo as P
    from paper_2502_08844_b200 import rollout as R
    from tests.conftest import GOLDEN

    g = np.load(os.path.join(GOLDEN, "evaluate_golden.npz"))
    with open(os.path.join(GOLDEN, "evaluate_golden.json")) as f:
        res = json.load(f)

    def check(got, want):
        assert got["eval_episode_steps"] == want["eval_episode_steps"]
        for k in ("eval_return_mean", "eval_return_std"):
            assert abs(got[k] - want[k]) <= 1e-5 * max(abs(want[k]), 1e-2), (k, got, want)

    policy = R.make_policy(5, 1, (32, 32)).cuda()
    policy.load_state_dict({k[4:]: torch.as_tensor(g[k]) for k in g.files if k.startswith("mlp/")})
    pn = P.DeviceRunningNormalizer(5, count=100.0, mean=g["pn/mean"], var=g["pn/var"])

    class Cfg:
        policy_obs_key = value_obs_key = "state"

    env = dk.DeviceBatchEnv(dk.EnvConfig(task="cartpole-balance", episode_length=25, seed=5), 32,
                            dtype="float64")
    check(R.evaluate_device(policy, env, Cfg, policy_normalizer=pn), res["mlp"][0])
    check(R.evaluate_device(policy, env, Cfg, max_steps=10, policy_normalizer=pn), res["mlp"][1])
    env.check()

    cnn = R.make_cnn_policy(3, 64, 1, (16,)).cuda()
    cnn.load_state_dict({k[4:]: torch.as_tensor(g[k]) for k in g.files if k.startswith("cnn/")})

    class PCfg:
        policy_obs_key, value_obs_key = "pixels", "state"

    penv = dk.DeviceBatchEnv(dk.EnvConfig(task="cartpole-balance-pixels", episode_length=6,
                                          visual_randomization=True, seed=2), 4, dtype="float64")
    tf32 = torch.backends.cudnn.allow_tf32
    torch.backends.cudnn.allow_tf32 = False
    try:
        check(R.evaluate_device(cnn, penv, PCfg), res["cnn"][0])
        check(R.evaluate_device(cnn, penv, PCfg), res["cnn"][1])
    finally:
        torch.backends.cudnn.allow_tf32 = tf32
    penv.check()


def test_go1_asymmetric_rollout_fused_equals_op_by_op():
    """The PPO rollout on the Go1 joystick env with an asymmetric actor-critic
    (policy on the noisy 56-wide observation, critic on the 75-wide privileged
    one, truncation bootstraps from the terminal privileged rows), both networks
    on the tensor cores: the fused bookkeeping kernels give bit-identical batch
    fields to the op-by-op torch path on an identically seeded env."""
    import paper_2502_08844_b200 as dk  # noqa: F401
    from paper_2502_08844_b200 import go1env as G
    from paper_2502_08844_b200 import ppo as P
    from paper_2502_08844_b200 import rollout as R

    class Cfg:
        unroll_length, reward_scaling, discounting = 8, 1.0, 0.99
        policy_obs_key, value_obs_key = "state", "privileged_state"

    torch.manual_seed(0)
    n = 300
    pol, val = R.make_policy(56, 12).cuda(), R.make_value(75).cuda()
    noise = torch.randn((Cfg.unroll_length, n, 12), device="cuda")
    res = []
    for op in (False, True):
        env = G.DeviceGo1Env(n, G.Go1Config(episode_length=5, term_height=0.22, seed=4))
        obs = env.reset(seed=4)
        pn, vn = P.DeviceRunningNormalizer(56), P.DeviceRunningNormalizer(75)
        pn.update(obs["state"])
        vn.update(obs["privileged_state"])
        batch, nxt, mr = R.collect_rollout_device(env, pol, val, Cfg, obs, pn, vn, noise=noise,
                                                  _op_by_op=op)
        env.check()
        res.append((batch, nxt, float(mr)))
        env.close()
    (b0, n0, m0), (b1, n1, m1) = res
    assert b0.dones.sum() > 0  # truncations inside the unroll: bootstraps exercised
    for f in ("policy_obs", "value_obs", "actions", "pre_tanh", "log_probs", "rewards", "dones",
              "values", "bootstrap", "raw_policy_obs", "raw_value_obs"):
        a, b = getattr(b0, f), getattr(b1, f)
        assert torch.equal(a.to(b.dtype), b), f
    assert torch.equal(n0["privileged_state"], n1["privileged_state"])
    assert abs(m0 - m1) < 1e-12 * max(1.0, abs(m1))


def test_go1_rollout_graph_replays():
    """RolloutGraph on the Go1 env (two static observation inputs; the env has
    no set_state, so the capture warm-up advances it one phase): replayed
    phases are finite, bootstrap through truncations, and match eager phases'
    shapes and dtypes."""
    from paper_2502_08844_b200 import go1env as G
    from paper_2502_08844_b200 import ppo as P
    from paper_2502_08844_b200 import rollout as R

    class Cfg:
        unroll_length, reward_scaling, discounting = 6, 1.0, 0.99
        policy_obs_key, value_obs_key = "state", "privileged_state"

    torch.manual_seed(1)
    env = G.DeviceGo1Env(200, G.Go1Config(episode_length=4, term_height=0.22, seed=6))
    obs = env.reset(seed=6)
    pol, val = R.make_policy(56, 12).cuda(), R.make_value(75).cuda()
    pn, vn = P.DeviceRunningNormalizer(56), P.DeviceRunningNormalizer(75)
    rg = R.RolloutGraph(env, pol, val, Cfg, obs, pn, vn)
    for _ in range(2):
        batch, nxt, mr = rg.run()
        for f in ("policy_obs", "value_obs", "actions", "log_probs", "rewards", "values",
                  "bootstrap"):
            assert torch.isfinite(getattr(batch, f)).all(), f
        assert batch.value_obs.shape == (6, 200, 75) and batch.policy_obs.shape == (6, 200, 56)
        assert batch.dones.sum() > 0
        assert nxt["privileged_state"].shape == (200, 75)
    env.close()
