"""The C oracle's PPO math against the reference's own outputs (CPU)."""
import os

import numpy as np
import pytest

from tests.conftest import GOLDEN


@pytest.fixture(scope="module")
def ppo_g():
    return np.load(os.path.join(GOLDEN, "ppo_golden.npz"))


@pytest.fixture(scope="module")
def orc():
    from oracle import ppo

    return ppo


@pytest.mark.parametrize("case", ["small", "mid"])
def test_gae_bit_exact(ppo_g, orc, case):
    g = lambda k: ppo_g[f"gae/{case}/{k}"]  # noqa: E731
    adv, ret = orc.gae(g("r"), g("v"), g("b"), g("d"), 0.97, 0.95)
    np.testing.assert_array_equal(adv, g("adv"))
    np.testing.assert_array_equal(ret, g("ret"))


def test_normalizer_bit_exact(ppo_g, orc):
    D = ppo_g["norm/probe"].shape[1]
    count, mean, var = 0.0, np.zeros(D), np.zeros(D)
    probe = ppo_g["norm/probe"]
    np.testing.assert_array_equal(orc.norm_apply(count, mean, var, 1e-8, probe),
                                  ppo_g["norm/apply0"])
    for k in range(3):
        count, mean, var = orc.norm_update(count, mean, var, ppo_g[f"norm/batch{k}"])
        assert count == float(ppo_g[f"norm/count{k}"])
        # NumPy reduces axis 0 of a C-contiguous array row by row: sequential sums
        np.testing.assert_array_equal(mean, ppo_g[f"norm/mean{k}"])
        np.testing.assert_array_equal(var, ppo_g[f"norm/var{k}"])
        np.testing.assert_array_equal(orc.norm_apply(count, mean, var, 1e-8, probe),
                                      ppo_g[f"norm/apply{k + 1}"])
        np.testing.assert_array_equal(orc.norm_apply(count, mean, var, 1e-8, probe, True),
                                      ppo_g[f"norm/invert{k + 1}"])


@pytest.mark.parametrize("case", ["stack", "const", "f32", "f64", "single"])
def test_pixel_normalize_bit_exact(orc, case):
    """ppo.pixel_normalize (ppo.py:232-238): sequential per-(sample, channel)
    sums reproduce NumPy's mean / std bit for bit, constant channels -> 0."""
    z = np.load(os.path.join(GOLDEN, "pixnorm_golden.npz"))
    np.testing.assert_array_equal(orc.pixel_normalize(z[f"{case}/x"]), z[f"{case}/y"])
