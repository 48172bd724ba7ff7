"""GPU parity of the locomotion step tail against the
reference's own outputs (tests/golden/loco_golden.npz) and the C oracle.

Tolerances: float64 -- 1e-12 relative (floor 1e-6): the kernels sum in the
reference's term order, NumPy's BLAS dot / pairwise sums / SIMD sin-cos differ
by ulps; selection, clipping, flags, Philox noise placement and integer logic
are exact.  float32 -- 1e-5 relative to max(|ref|, floor_col): per output
column, floor_col = max(1e-6, K * E_col / 1e-5) (K = 4, tests/f32_envelope.py)
where E_col is how far the float64 oracle's output moves when its input frame
and its output are rounded to float32 -- the deviation any float32
implementation inherits (cancellations such as command - velocity amplify the
input rounding); a column unaffected by rounding keeps the 1e-6 floor.
"""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GATED = dict(standstill_gated=True, w_lin_vel=1.5, sigma_phase=0.01, w_energy=-2e-3,
             airtime_min=0.05, airtime_max=0.4)


@pytest.fixture(scope="module")
def loco():
    from tests.conftest import GOLDEN

    return np.load(os.path.join(GOLDEN, "loco_golden.npz"))


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2502_08844_b200 import locomotion

    return locomotion


def _frames(loco, shape, dtype):
    out = {}
    for k in loco.files:
        if k.startswith(f"{shape}/frame/"):
            v = loco[k]
            name = k.split("/")[-1]
            t = torch.as_tensor(v, device="cuda")
            out[name] = t if v.dtype == np.uint8 else t.to(dtype)
    return out


def _close(a, b, floor):
    a = a.double().cpu().numpy() if hasattr(a, "cpu") else np.asarray(a, float)
    b = np.asarray(b, float)
    return float((np.abs(a - b) / np.maximum(np.abs(b), floor)).max())


TOL = {torch.float64: (1e-12, 1e-6), torch.float32: (1e-5, None)}


def _np_frames(loco, shape):
    return {k.split("/")[-1]: loco[k] for k in loco.files if k.startswith(f"{shape}/frame/")}


def _r32(x):
    return np.asarray(x).astype(np.float32).astype(np.float64) if np.asarray(x).dtype.kind == "f" \
        else np.asarray(x)


def _f32_floor(fn, frames):
    """per-column floors from the float32 rounding of the inputs and outputs"""
    from tests.f32_envelope import K_ULP

    exact = np.asarray(fn(frames), np.float64)
    rounded = _r32(np.asarray(fn({k: _r32(v) for k, v in frames.items()}), np.float64))
    E = np.abs(rounded - exact)
    E = E.max(axis=0) if E.ndim > 1 else E.max()
    return np.maximum(1e-6, K_ULP * E / 1e-5)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("shape", ["go1", "biped"])
@pytest.mark.parametrize("cfg", ["default", "gated"])
def test_total_reward_matches_reference(loco, L, dtype, shape, cfg):
    fr = _frames(loco, shape, dtype)
    c = L.RewardTermConfig(**({} if cfg == "default" else GATED))
    br = L.total_reward_batch(fr, c)
    tol, floor = TOL[dtype]
    g = lambda k: loco[f"{shape}/reward/{cfg}/{k}"]  # noqa: E731
    terms = torch.stack([br.terms[n] for n in L.TERM_NAMES], 1)
    fl = [floor] * 3
    if floor is None:
        from oracle import locomotion as olo

        kw = {} if cfg == "default" else GATED
        nf = _np_frames(loco, shape)
        fl = [_f32_floor(lambda f, i=i: olo.total_reward(f, **kw)[i], nf) for i in range(3)]
        np.testing.assert_allclose(olo.total_reward(nf, **kw)[0], g("terms"), rtol=1e-12,
                                   atol=1e-12)  # the oracle is pinned on these frames
    assert _close(terms, g("terms"), fl[0]) < tol
    assert _close(br.unclipped_total, g("unclipped"), fl[1]) < tol
    assert _close(br.total, g("total"), fl[2]) < tol
    if dtype == torch.float64:
        np.testing.assert_array_equal(br.total.cpu().numpy() == 0.0, g("total") == 0.0)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("shape", ["go1", "biped"])
@pytest.mark.parametrize("kind", ["noisy", "partial", "clean"])
def test_observation_matches_reference(loco, L, dtype, shape, kind):
    fr = _frames(loco, shape, dtype)
    nz = {"noisy": loco["obs/noise"], "partial": loco["obs/partial_noise"], "clean": None}[kind]
    noise = None if nz is None else L.ObservationNoise(*[float(x) for x in nz])
    seed, env0, ep, step = (int(x) for x in loco["obs/key"])
    n = fr["joint_pos"].shape[0]
    key = L.NoiseKey(seed, env0, torch.full((n,), ep, device="cuda"), step)
    pert = None if kind == "clean" else torch.as_tensor(loco[f"{shape}/obs/pert"], device="cuda")
    o = L.build_locomotion_observation_batch(fr, fr["prev_action"], fr["command"], noise, key,
                                             pert)
    tol, floor = TOL[dtype]
    fs = fp = floor
    if floor is None:
        from oracle import locomotion as olo

        nf = _np_frames(loco, shape)
        pn = None if pert is None else pert.cpu().numpy()
        nzl = None if noise is None else [float(x) for x in nz]

        def obs(f, i):
            return olo.loco_obs(f, f["prev_action"], f["command"], nzl, (seed, env0, ep, step),
                                pn)[i]

        fs, fp = _f32_floor(lambda f: obs(f, 0), nf), _f32_floor(lambda f: obs(f, 1), nf)
    assert _close(o["state"], loco[f"{shape}/obs/{kind}/state"], fs) < tol
    assert _close(o["privileged_state"], loco[f"{shape}/obs/{kind}/priv"], fp) < tol


def test_fused_tail_large_batch_vs_oracle(loco, L, oracle):
    """8192 worlds x 4 steps (Go1 shape) vs the C oracle, incl. the per-step
    Philox noise streams (step-major rows)."""
    from oracle import locomotion as olo

    src = {k.split("/")[-1]: loco[k] for k in loco.files if k.startswith("go1/frame/")}
    n0 = src["joint_pos"].shape[0]
    N, K = 8192, 4
    idx = np.random.default_rng(0).integers(0, n0, K * N)
    big = {k: v[idx] for k, v in src.items()}
    jit = np.random.default_rng(1).normal(0, 0.01, big["joint_pos"].shape)
    big["joint_pos"] = big["joint_pos"] + jit
    noise = [0.05, 0.1, 0.2, 0.01, 1.5]
    tr = torch.as_tensor
    fr = {k: tr(v, device="cuda") for k, v in big.items()}
    out = L.locomotion_tail(fr, L.RewardTermConfig(), noise=L.ObservationNoise(*noise),
                            key=L.NoiseKey(3, 100, None, 7), num_worlds=N)
    terms, unc, tot, bad = olo.total_reward(big)
    assert bad == -1
    assert _close(out["terms"], terms, 1e-6) < 1e-12
    assert _close(out["total"], tot, 1e-6) < 1e-12
    for k in range(K):
        rows = slice(k * N, (k + 1) * N)
        sub = {f: v[rows] for f, v in big.items()}
        st, pr, _ = olo.loco_obs(sub, noise=noise, key=(3, 100, 0, 7 + k))
        assert _close(out["state"][rows], st, 1e-6) < 1e-12
        assert _close(out["privileged_state"][rows], pr, 1e-6) < 1e-12


def test_non_unit_quaternion_raises(loco, L):
    fr = _frames(loco, "go1", torch.float64)
    fr["base_orientation"] = fr["base_orientation"].clone()
    fr["base_orientation"][5] *= 1.0 + 2e-6
    with pytest.raises(L.InvalidInputError, match="quaternion is not unit length"):
        L.locomotion_tail(fr)


@pytest.mark.parametrize("mode", ["abs", "rel"])
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_pd(loco, L, mode, dtype):
    kp, kd, sc, lim, lo, hi, rel = loco[f"pd/{mode}/params"]
    p = L.PDParams(kp, kd, sc, loco["pd/qdef"], mode="relative" if rel else "absolute",
                   torque_limit=lim, joint_range=(lo, hi))
    t = lambda k: torch.as_tensor(loco[k], device="cuda", dtype=dtype)  # noqa: E731
    tgt, tau = L.pd_batch(t("pd/a"), t("pd/prev"), t("pd/q"), t("pd/v"), p)
    if dtype == torch.float64:
        np.testing.assert_array_equal(tgt.cpu().numpy(), loco[f"pd/{mode}/target"])
        np.testing.assert_array_equal(tau.cpu().numpy(), loco[f"pd/{mode}/torque"])
    else:  # kp (up to 35) amplifies the float32 rounding of the inputs
        from oracle import locomotion as olo

        ins = {k: loco[f"pd/{k}"] for k in ("a", "prev", "q", "v")}
        prm = loco[f"pd/{mode}/params"]
        fn = lambda f: olo.pd(prm, loco["pd/qdef"], f["a"], f["prev"], f["q"], f["v"])  # noqa: E731
        np.testing.assert_array_equal(fn(ins)[1], loco[f"pd/{mode}/torque"])  # pinned oracle
        assert _close(tgt, loco[f"pd/{mode}/target"], _f32_floor(lambda f: fn(f)[0], ins)) < 1e-5
        assert _close(tau, loco[f"pd/{mode}/torque"], _f32_floor(lambda f: fn(f)[1], ins)) < 1e-5


def test_phase_and_progress(loco, L):
    t = lambda k: torch.as_tensor(loco[k], device="cuda")  # noqa: E731
    phi, cs = L.advance_phase_batch(t("phase/phi"), t("phase/freq"), t("phase/dt"))
    assert _close(phi, loco["phase/advanced"], 1e-9) < 1e-14
    p0, cs0 = L.advance_phase_batch(t("phase/phi"), 0.0, 0.0)  # wrap only
    assert _close(cs0.reshape(cs0.shape[0], -1), loco["phase/encoded"].reshape(cs0.shape[0], -1),
                  1e-6) < 1e-14
    r, h = L.progress_clip_reward_batch(t("progress/raw"), t("progress/hist"))
    np.testing.assert_array_equal(torch.stack([r, h], 1).cpu().numpy(), loco["progress/out"])


def test_dr_primitives(loco, L):
    class Spec:
        def __init__(self, slot, scale):
            self.slot, self.scale, self.kind = slot, scale, "uniform"

    x = torch.as_tensor(loco["dr/noise_in"], device="cuda")
    obs = {"a": x[:, :3], "b": x[:, 3:6], "c": x[:, 6:]}
    out = L.apply_sensor_noise_batch(obs, [Spec("a", 0.1), Spec("b", 0.0), Spec("c", 0.5)],
                                     L.NoiseKey(5, 0, None, 1))
    got = torch.cat([out["a"], out["b"], out["c"]], 1).cpu().numpy()
    np.testing.assert_array_equal(got, loco["dr/noise_out"])
    with pytest.raises(L.ConfigError):
        L.apply_sensor_noise_batch(obs, [Spec("privileged_state", 0.1)], L.NoiseKey())
    pose, inj = L.pose_injection_batch(torch.as_tensor(loco["dr/pose_in"], device="cuda"), 0.4,
                                       loco["dr/pose_bounds"],
                                       L.NoiseKey(9, 0, torch.full((64,), 3, device="cuda"), 0))
    np.testing.assert_array_equal(pose.cpu().numpy(), loco["dr/pose_out"])
    seq = torch.as_tensor(loco["dr/curr_seq"], device="cuda")
    st = torch.zeros((seq.shape[0], 4), dtype=torch.int64, device="cuda")
    hist = []
    for k in range(seq.shape[1]):
        st = L.curriculum_update_batch(st, seq[:, k], max_level=5, promotion_threshold=2)
        hist.append(st)
    np.testing.assert_array_equal(torch.stack(hist, 1).cpu().numpy(), loco["dr/curr_out"])


class _Spec:
    def __init__(self, slot, scale, kind="uniform"):
        self.slot, self.scale, self.kind = slot, scale, kind


def test_gaussian_sensor_noise(loco, L):
    # Generator.normal through NumPy's ziggurat on the GPU: bit-exact in f64
    x = torch.as_tensor(loco["dr/gnoise_in"], device="cuda")
    obs = {"a": x[:, :4], "b": x[:, 4:6], "c": x[:, 6:]}
    specs = [_Spec("a", 0.2, "gaussian"), _Spec("b", 0.05), _Spec("c", 1.5, "gaussian")]
    out = L.apply_sensor_noise_batch(obs, specs, L.NoiseKey(6, 100, torch.full((48,), 1,
                                                                            device="cuda"), 7))
    got = torch.cat([out["a"], out["b"], out["c"]], 1).cpu().numpy()
    np.testing.assert_array_equal(got, loco["dr/gnoise_out"])
    # f32 rows: the same draws, added in f64 and rounded once
    o32 = L.apply_sensor_noise_batch({k: v.float() for k, v in obs.items()}, specs,
                                     L.NoiseKey(6, 100, torch.full((48,), 1, device="cuda"), 7))
    g32 = torch.cat([o32["a"], o32["b"], o32["c"]], 1).double().cpu().numpy()
    # within the float32 rounding of the input plus that of the result (2 ulp)
    ref = loco["dr/gnoise_out"]
    xin = x.cpu().numpy()
    ulp = np.spacing(np.maximum(np.abs(ref), np.abs(xin)).astype(np.float32)).astype(np.float64)
    assert (np.abs(g32 - ref) <= 2 * ulp).all()
    with pytest.raises(L.ConfigError):
        L.apply_sensor_noise_batch(obs, [_Spec("a", 0.1, "laplace")], L.NoiseKey())


def test_gaussian_noise_many_streams_vs_oracle(L):
    # 65536 worlds x 32 gaussian draws (wedge and tail paths hit ~2000 times)
    from oracle import locomotion as orc

    n, d = 65536, 32
    x = torch.zeros((n, d), dtype=torch.float64, device="cuda")
    out = L.apply_sensor_noise_batch({"s": x}, [_Spec("s", 1.0, "gaussian")],
                                     L.NoiseKey(1234, 7, None, 3))["s"].cpu().numpy()
    ref = orc.sensor_noise(np.zeros((n, d)), [(0, d, 1.0, "gaussian")], key=(1234, 7, 0, 3))
    # identical draw sequence; the tail's log1p (CUDA vs glibc) may differ by an
    # ulp (measured: 4 of 2M values, 1 ulp), every other path is bit-exact
    np.testing.assert_allclose(out, ref, rtol=1e-15, atol=0)
    assert np.count_nonzero(out != ref) <= 64


def test_randomize_params(loco, L):
    import dataclasses

    names = [str(s) for s in loco["dr/params_fields"]]

    @dataclasses.dataclass
    class Nominal:
        pass

    Nom = dataclasses.make_dataclass("Nom", [(k, float) for k in names])
    nominal = Nom(*[float(v) for v in loco["dr/params_nominal"]])

    class PR:
        def __init__(self, path, dist, lo, hi):
            self.path, self.distribution, self.low, self.high = path, dist, lo, hi

    dists = ("uniform_additive", "uniform_multiplicative", "log_uniform")
    spec = type("Spec", (), {"params": tuple(PR(names[int(r[0])], dists[int(r[1])], r[2], r[3])
                                             for r in loco["dr/params_ranges"])})()
    out, fields = L.randomize_params_batch(nominal, spec, L.NoiseKey(21, 0, torch.full(
        (64,), 4, device="cuda"), 0), 64)
    assert fields == names
    # NumPy's SIMD exp vs CUDA exp on the log-uniform field: a few ulps
    np.testing.assert_allclose(out.cpu().numpy(), loco["dr/params_out"], rtol=1e-14, atol=0)
    bad = type("Spec", (), {"params": (PR("pend_mass", "uniform_additive", -9, -5),)})()
    with pytest.raises(L.ConfigError, match="pend_mass"):
        L.randomize_params_batch(nominal, bad, L.NoiseKey(21, 0, None, 0), 8)
    with pytest.raises(L.ConfigError):
        L.randomize_params_batch(nominal, type("S", (), {"params": (PR("nope", dists[0], 0, 1),)})(),
                                 L.NoiseKey(), 4)


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_delay_lines(loco, L, dtype):
    tdt = getattr(torch, dtype)
    vals = torch.as_tensor(loco["dr/delay_in"], device="cuda", dtype=tdt)  # [24, 16, 3]
    for mode, (lo, hi, per_step) in (("ep", (1, 3, False)), ("st", (0, 5, True))):
        dl = L.DelayLineBatch(16, 3, lo, hi, per_step, dtype=tdt)
        ep = torch.full((16,), 2, device="cuda")
        dl.reset(L.NoiseKey(31, 0, ep, 0))
        np.testing.assert_array_equal(dl.delay.cpu().numpy(), loco[f"dr/delay_{mode}_delay"])
        outs = torch.stack([dl.push_pop(vals[t], L.NoiseKey(32, 0, ep, t))
                            for t in range(vals.shape[0])])
        np.testing.assert_array_equal(outs.double().cpu().numpy(),
                                      loco[f"dr/delay_{mode}_out"].astype(dtype).astype(np.float64))
    with pytest.raises(L.ConfigError):
        L.DelayLineBatch(4, 1, 3, 2)
    with pytest.raises(L.ConfigError):
        L.DelayLineBatch(4, 1, 0, 2).push_pop(torch.zeros(4, 1, device="cuda"))
