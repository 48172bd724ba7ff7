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
