"""GPU PPO math (compute_gae, RunningNormalizer) against the reference's outputs
(tests/golden/ppo_golden.npz) and the C oracle.

GAE and normalizer apply / invert are float64 in the reference's operation order:
bit-exact.  normalizer_update sums each column as a fixed-order tree where NumPy
sums rows sequentially: mean / var agree to 1e-13 relative (stated tolerance).
float32 storage: the same float64 arithmetic on the f32 inputs, rounded once."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ppo_g():
    from tests.conftest import GOLDEN

    return np.load(os.path.join(GOLDEN, "ppo_golden.npz"))


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2502_08844_b200 import ppo

    return ppo


def _t(a, dt=torch.float64):
    return torch.as_tensor(np.asarray(a), device="cuda").to(dt)


@pytest.mark.parametrize("case", ["small", "mid"])
def test_gae_matches_reference(ppo_g, P, case):
    g = lambda k: ppo_g[f"gae/{case}/{k}"]  # noqa: E731
    adv, ret = P.compute_gae_batch(_t(g("r")), _t(g("v")), _t(g("b")), _t(g("d")), 0.97, 0.95)
    np.testing.assert_array_equal(adv.cpu().numpy(), g("adv"))
    np.testing.assert_array_equal(ret.cpu().numpy(), g("ret"))


def test_gae_float32_and_large_vs_oracle(P):
    from oracle import ppo as orc

    rng = np.random.default_rng(7)
    T, N = 1000, 8192
    r = rng.normal(0, 1, (T, N)).astype(np.float32)
    v = rng.normal(0, 1, (T, N)).astype(np.float32)
    d = (rng.uniform(size=(T, N)) < 0.001).astype(np.float32)
    b = rng.normal(0, 1, N).astype(np.float32)
    adv, ret = P.compute_gae_batch(_t(r, torch.float32), _t(v, torch.float32),
                                   _t(b, torch.float32), _t(d, torch.float32), 0.99, 0.95)
    ra, rr = orc.gae(r, v, b, d, 0.99, 0.95)
    np.testing.assert_array_equal(adv.cpu().numpy(), ra.astype(np.float32))
    np.testing.assert_array_equal(ret.cpu().numpy(), rr.astype(np.float32))
    with pytest.raises(P.InvalidInputError):
        P.compute_gae_batch(_t(r[:, :3]), _t(v[:, :4]), _t(b[:3]), _t(d[:, :3]), 0.99, 0.95)


def test_normalizer_matches_reference(ppo_g, P):
    probe = ppo_g["norm/probe"]
    D = probe.shape[1]
    n = P.DeviceRunningNormalizer(D)
    np.testing.assert_array_equal(n.apply(_t(probe)).cpu().numpy(), ppo_g["norm/apply0"])
    for k in range(3):
        n.update(_t(ppo_g[f"norm/batch{k}"]))
        c, m, v = n.to_numpy()
        assert c == float(ppo_g[f"norm/count{k}"])
        np.testing.assert_allclose(m, ppo_g[f"norm/mean{k}"], rtol=1e-13, atol=1e-15)
        np.testing.assert_allclose(v, ppo_g[f"norm/var{k}"], rtol=1e-13, atol=1e-15)
        # apply / invert on the reference's own statistics: bit-exact
        ref = P.DeviceRunningNormalizer(D, count=c, mean=ppo_g[f"norm/mean{k}"],
                                        var=ppo_g[f"norm/var{k}"])
        np.testing.assert_array_equal(ref.apply(_t(probe)).cpu().numpy(),
                                      ppo_g[f"norm/apply{k + 1}"])
        np.testing.assert_array_equal(ref.invert(_t(probe)).cpu().numpy(),
                                      ppo_g[f"norm/invert{k + 1}"])
        # f32 storage: f64 arithmetic rounded once
        np.testing.assert_array_equal(ref.apply(_t(probe, torch.float32)).cpu().numpy(),
                                      _apply_ref32(probe, c, ppo_g, k))
    with pytest.raises(P.InvalidInputError):
        n.update(_t(probe[:, :3]))


def _apply_ref32(probe, c, ppo_g, k):
    from oracle import ppo as orc

    x32 = probe.astype(np.float32).astype(np.float64)
    return orc.norm_apply(c, ppo_g[f"norm/mean{k}"], ppo_g[f"norm/var{k}"], 1e-8,
                          x32).astype(np.float32)


def test_normalizer_large_vs_oracle(P):
    from oracle import ppo as orc

    rng = np.random.default_rng(11)
    x = rng.normal(rng.uniform(-3, 3, 75), rng.uniform(0.01, 4, 75), (1000 * 64, 75))
    n = P.DeviceRunningNormalizer(75)
    n.update(_t(x.astype(np.float32)))
    n.update(_t(x[:777]))
    c, m, v = orc.norm_update(0.0, np.zeros(75), np.zeros(75),
                              x.astype(np.float32).astype(np.float64))
    c, m, v = orc.norm_update(c, m, v, x[:777])
    gc, gm, gv = n.to_numpy()
    assert gc == c
    np.testing.assert_allclose(gm, m, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(gv, v, rtol=1e-12)


@pytest.mark.parametrize("dt", ["float32", "float64"])
@pytest.mark.parametrize("T,N", [(77, 36), (1, 4), (64, 100), (33, 8)])
def test_gae_ragged_vs_oracle(P, dt, T, N):
    """GAE on ragged shapes (T not a multiple of the kernel's 16-step register
    chunks, partial 128-world blocks, frequent terminations), both dtypes;
    bit-exact against the oracle."""
    from oracle import ppo as orc

    npdt = np.float32 if dt == "float32" else np.float64
    tdt = torch.float32 if dt == "float32" else torch.float64
    rng = np.random.default_rng(T * 1000 + N)
    r = rng.normal(0, 1, (T, N)).astype(npdt)
    v = rng.normal(0, 1, (T, N)).astype(npdt)
    d = (rng.uniform(size=(T, N)) < 0.05).astype(npdt)
    b = rng.normal(0, 1, N).astype(npdt)
    adv, ret = P.compute_gae_batch(_t(r, tdt), _t(v, tdt), _t(b, tdt), _t(d, tdt), 0.99, 0.95)
    ra, rr = orc.gae(r, v, b, d, 0.99, 0.95)
    np.testing.assert_array_equal(adv.cpu().numpy(), ra.astype(npdt))
    np.testing.assert_array_equal(ret.cpu().numpy(), rr.astype(npdt))


def test_step_post_equals_separate_kernels():
    """dk_ppo_step_post == dk_ppo_step_bootstrap_acc + dk_ppo_step_record (values /
    term_values NULL) + dk_ppo_step_inputs, and the deferred reward targets
    (record without term_values, then dk_ppo_boot_fixup) == the direct ones,
    bit for bit; slots keep counting across calls (the boot rows' slot order
    follows the atomics, so rows are compared through pos)."""
    import ctypes

    from paper_2502_08844_b200 import _native as nat

    lib = nat.lib()
    g = torch.Generator(device="cuda").manual_seed(3)
    N, dp, dv, A = 1000, 7, 9, 3
    u8 = lambda p: (torch.rand(N, device="cuda", generator=g) < p).to(torch.uint8)  # noqa: E731
    rn = lambda *s: torch.randn(*s, device="cuda", generator=g)  # noqa: E731
    done, trunc, tmask = u8(0.1), u8(0.3), u8(0.8)
    term_obs, reward, action = rn(N, dv), rn(N), rn(N, A)
    obs_p, obs_v = rn(N, dp), rn(N, dv)
    mk = lambda d: (torch.rand(d, device="cuda", dtype=torch.float64, generator=g),  # noqa: E731
                    torch.rand(d, device="cuda", dtype=torch.float64, generator=g) + 0.5)
    (mp, vp), (mv, vv) = mk(dp), mk(dv)
    norm_p = nat.PpoNormC(mp.data_ptr(), vp.data_ptr(), 1e-8, 0, 1)
    norm_v = nat.PpoNormC(mv.data_ptr(), vv.data_ptr(), 1e-8, 0, 1)
    scale, disc = 0.3, 0.97
    nb = int(lib.dk_ppo_record_blocks(N))

    def bufs():
        z = lambda *s, d=torch.float32: torch.zeros(*s, dtype=d, device="cuda")  # noqa: E731
        return dict(vterm=z(2 * N, dv), count=z(1, d=torch.int64), pos=z(N, d=torch.int32),
                    dones=z(N, d=torch.float64), rew=z(N, d=torch.float64),
                    acts=z(N, A, d=torch.float64), part=z(nb, d=torch.float64),
                    rawp=z(N, dp), rawv=z(N, dv), pol=z(N, dp), val=z(N, dv))

    a, b = bufs(), bufs()
    for x in (a, b):
        x["count"].fill_(5)  # slots continue from earlier steps of the phase
    P = lambda t: t.data_ptr()  # noqa: E731
    assert lib.dk_ppo_step_bootstrap_acc(
        N, dv, P(done), P(trunc), P(tmask), P(term_obs), ctypes.byref(norm_v), P(a["vterm"]),
        P(a["count"]), P(a["pos"]), P(a["dones"]), None) == 0
    assert lib.dk_ppo_step_record(
        N, A, P(reward), P(a["pos"]), None, None, P(action), scale, disc, P(a["rew"]), None,
        P(a["acts"]), P(a["part"]), None) == 0
    assert lib.dk_ppo_step_inputs(
        N, dp, dv, P(obs_p), P(obs_v), ctypes.byref(norm_p), ctypes.byref(norm_v), P(a["rawp"]),
        P(a["rawv"]), P(a["pol"]), P(a["val"]), None, None) == 0
    post = nat.PpoPostC(
        n=N, dp=dp, dv=dv, action_dim=A, done=P(done), trunc=P(trunc), terminal_mask=P(tmask),
        terminal_obs=P(term_obs), val_term=P(b["vterm"]), count=P(b["count"]), pos=P(b["pos"]),
        dones=P(b["dones"]), reward=P(reward), action=P(action), reward_scaling=scale,
        discounting=disc, rewards_out=P(b["rew"]), actions_out=P(b["acts"]),
        reward_partial=P(b["part"]), next_obs_p=P(obs_p), next_obs_v=P(obs_v),
        next_raw_p=P(b["rawp"]), next_raw_v=P(b["rawv"]), next_pol=P(b["pol"]),
        next_val=P(b["val"]))
    assert lib.dk_ppo_step_post(ctypes.byref(post), ctypes.byref(norm_p), ctypes.byref(norm_v),
                                None) == 0
    torch.cuda.synchronize()
    boot = (trunc.bool() & ~done.bool() & tmask.bool())
    assert int(a["count"]) == int(b["count"]) == 5 + int(boot.sum()) and boot.sum() > 10
    for k in ("dones", "rew", "acts", "part", "rawp", "rawv", "pol", "val"):
        assert torch.equal(a[k], b[k]), k
    assert torch.equal(a["pos"] >= 0, boot) and torch.equal(b["pos"] >= 0, boot)
    ia, ib = a["pos"][boot].long(), b["pos"][boot].long()
    assert torch.equal(a["vterm"][ia], b["vterm"][ib]) and int(ia.min()) >= 5

    # deferred reward targets == direct ones
    tv = rn(2 * N)
    direct = torch.zeros(N, dtype=torch.float64, device="cuda")
    part = torch.zeros(nb, dtype=torch.float64, device="cuda")
    acts = torch.zeros(N, A, dtype=torch.float64, device="cuda")
    assert lib.dk_ppo_step_record(
        N, A, P(reward), P(a["pos"]), None, P(tv), P(action), scale, disc, P(direct), None,
        P(acts), P(part), None) == 0
    assert lib.dk_ppo_boot_fixup(N, P(a["pos"]), P(tv), disc, P(a["rew"]), None) == 0
    torch.cuda.synchronize()
    assert torch.equal(direct, a["rew"])
