"""Pin the locomotion-tail oracle (oracle/locomotion.c) to the reference.

Fixtures: tests/golden/loco_golden.npz from tests/golden/make_golden_loco.py
(the reference itself).  Selection, clipping, flags, counters and Philox noise
placement are compared exactly; floating sums to 1e-12 relative (NumPy's BLAS
dot / pairwise sums / SIMD sin-cos reassociate the reference's arithmetic).
"""

import numpy as np
import pytest

RTOL = 1e-12


@pytest.fixture(scope="module")
def loco():
    import os

    from tests.conftest import GOLDEN

    return np.load(os.path.join(GOLDEN, "loco_golden.npz"))


@pytest.fixture(scope="module")
def orc(oracle):
    from oracle import locomotion

    return locomotion


def _frames(loco, shape):
    return {k.split("/")[-1]: loco[k] for k in loco.files if k.startswith(f"{shape}/frame/")}


def _close(a, b, rtol=RTOL, floor=1e-9):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float((np.abs(a - b) / np.maximum(np.abs(b), floor)).max())


GATED = dict(standstill_gated=True, w_lin_vel=1.5, sigma_phase=0.01, w_energy=-2e-3,
             airtime_min=0.05, airtime_max=0.4)


@pytest.mark.parametrize("shape", ["go1", "biped"])
@pytest.mark.parametrize("cfg", ["default", "gated"])
def test_total_reward(loco, orc, shape, cfg):
    fr = _frames(loco, shape)
    terms, unc, tot, bad = orc.total_reward(fr, **({} if cfg == "default" else GATED))
    assert bad == -1
    g = lambda k: loco[f"{shape}/reward/{cfg}/{k}"]  # noqa: E731
    assert _close(terms, g("terms")) < RTOL
    assert _close(unc, g("unclipped"), floor=1e-6) < RTOL
    assert _close(tot, g("total"), floor=1e-6) < RTOL
    np.testing.assert_array_equal(tot == 0.0, g("total") == 0.0)  # the non-negative clip


@pytest.mark.parametrize("shape", ["go1", "biped"])
@pytest.mark.parametrize("kind", ["noisy", "partial", "clean"])
def test_locomotion_observation(loco, orc, shape, kind):
    fr = _frames(loco, shape)
    noise = {"noisy": loco["obs/noise"], "partial": loco["obs/partial_noise"], "clean": None}[kind]
    seed, env0, ep, step = (int(x) for x in loco["obs/key"])
    st, pr, bad = orc.loco_obs(fr, noise=noise, key=(seed, env0, ep, step),
                               pert=None if kind == "clean" else loco[f"{shape}/obs/pert"])
    assert bad == -1
    assert st.shape == loco[f"{shape}/obs/{kind}/state"].shape
    assert _close(st, loco[f"{shape}/obs/{kind}/state"], floor=1e-6) < RTOL
    assert _close(pr, loco[f"{shape}/obs/{kind}/priv"], floor=1e-6) < RTOL


def test_project_gravity(loco, orc):
    out, ok = orc.project_gravity(loco["gravity/q"])
    assert ok.all()
    assert _close(out, loco["gravity/out"], floor=1e-6) < RTOL
    _, ok = orc.project_gravity(loco["gravity/bad_q"])
    np.testing.assert_array_equal(ok, loco["gravity/bad_ok"])


def test_phase(loco, orc):
    np.testing.assert_array_equal(orc.wrap_angle(loco["phase/wrap_in"]), loco["phase/wrap_out"])
    adv = orc.advance_phase(loco["phase/phi"], loco["phase/freq"], loco["phase/dt"])
    assert _close(adv, loco["phase/advanced"], floor=1e-9) < 1e-14


@pytest.mark.parametrize("mode", ["abs", "rel"])
def test_pd(loco, orc, mode):
    tgt, tau = orc.pd(loco[f"pd/{mode}/params"], loco["pd/qdef"], loco["pd/a"], loco["pd/prev"],
                      loco["pd/q"], loco["pd/v"])
    np.testing.assert_array_equal(tgt, loco[f"pd/{mode}/target"])
    np.testing.assert_array_equal(tau, loco[f"pd/{mode}/torque"])


def test_progress_clip(loco, orc):
    r, h = orc.progress_clip(loco["progress/raw"], loco["progress/hist"])
    np.testing.assert_array_equal(np.stack([r, h], 1), loco["progress/out"])


def test_sensor_noise_and_pose_injection(loco, orc):
    specs = [(0, 3, 0.1), (3, 3, 0.0), (6, 3, 0.5)]
    out = orc.sensor_noise(loco["dr/noise_in"], specs, key=(5, 0, 0, 1))
    np.testing.assert_array_equal(out, loco["dr/noise_out"])
    inj = orc.pose_injection(loco["dr/pose_in"], loco["dr/pose_bounds"], 0.4, key=(9, 0, 3, 0))
    np.testing.assert_array_equal(inj, loco["dr/pose_out"])


def test_gaussian_sensor_noise(loco, orc):
    # Generator.normal through NumPy's ziggurat: bit-exact
    specs = [(0, 4, 0.2, "gaussian"), (4, 2, 0.05, "uniform"), (6, 4, 1.5, "gaussian")]
    out = orc.sensor_noise(loco["dr/gnoise_in"], specs, key=(6, 100, 1, 7))
    np.testing.assert_array_equal(out, loco["dr/gnoise_out"])


def test_stream_normal_and_integers_known_answers(loco, orc):
    # Generator.standard_normal (4096 draws: ~15 take the wedge / tail paths) and
    # Generator.integers (32-bit Lemire with the half-word buffer), bit-exact
    np.testing.assert_array_equal(orc.stream_normal((0, 0, 0, 0), 4096), loco["dr/normal_known"])
    got = orc.stream_integers((0, 0, 0, 0), 1, 4, 64)
    np.testing.assert_array_equal(got, loco["dr/int_known"][:64])


def test_randomize_params(loco, orc):
    ranges = [(int(r[0]), ("uniform_additive", "uniform_multiplicative", "log_uniform")[int(r[1])],
               r[2], r[3]) for r in loco["dr/params_ranges"]]
    out, fail = orc.randomize_params(loco["dr/params_nominal"], ranges, 64, key=(21, 0, 4, 0))
    assert fail == -1
    # NumPy's exp/log ufuncs (SIMD) vs glibc: a few ulps on the log-uniform field
    np.testing.assert_allclose(out, loco["dr/params_out"], rtol=1e-14, atol=0)
    # a field that can never be drawn positive -> the first world fails (ConfigError)
    _, fail = orc.randomize_params(loco["dr/params_nominal"], [(2, "uniform_additive", -9, -5)],
                                   8, key=(21, 0, 4, 0))
    assert fail == 0


def test_delay_lines(loco, orc):
    vals = loco["dr/delay_in"]
    for mode, (lo, hi, per_step) in (("ep", (1, 3, False)), ("st", (0, 5, True))):
        dl = orc.DelayLines(16, 3, lo, hi, per_step)
        dl.reset((31, 0, 2, 0))
        np.testing.assert_array_equal(dl.delay, loco[f"dr/delay_{mode}_delay"])
        outs = np.stack([dl.push_pop(vals[t], (32, 0, 2, t)) for t in range(vals.shape[0])])
        np.testing.assert_array_equal(outs, loco[f"dr/delay_{mode}_out"])


def test_curriculum(loco, orc):
    seq = loco["dr/curr_seq"]
    st = np.zeros((seq.shape[0], 4), dtype=np.int64)
    hist = []
    for t in range(seq.shape[1]):
        st = orc.curriculum(st, seq[:, t], max_level=5, threshold=2)
        hist.append(st.copy())
    np.testing.assert_array_equal(np.stack(hist, 1), loco["dr/curr_out"])
