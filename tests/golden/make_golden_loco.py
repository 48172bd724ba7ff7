"""Golden fixtures for the locomotion step tail,
generated from the REFERENCE (deskrl 0.1.0) in the build container:

    python tests/golden/make_golden_loco.py

Covers rewards.total_reward + the 16 terms (rewards.py:97-211), envkit.
build_locomotion_observation with Philox-keyed uniform noise (envkit.py:147-193),
mathcore.project_gravity / quat_check_unit (mathcore.py:42-97), wrap_angle /
advance_phase / phase_encode (mathcore.py:143-177), swing_height_profile
(rewards.py:92-94), action_to_target / pd_torque (envkit.py:111-131),
progress_clip_reward (envkit.py:196-202), randomization.apply_sensor_noise
(uniform, randomization.py:88-108), pose_injection (188-199) and
curriculum_update (224-238).  Frames come from gaitgen.random_frame and
GaitGenerator (gaitgen.py:31-129) at Go1 shape (12 joints, 4 feet) and the
gaitgen default shape (8 joints, 2 feet).
"""

from __future__ import annotations

import dataclasses
import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))

FIELDS = ["base_orientation", "base_lin_vel", "base_ang_vel", "joint_pos", "joint_vel",
          "joint_torque", "foot_height", "foot_height_des", "foot_vel_xy", "foot_contact",
          "airtime", "touchdown", "phase", "command", "action", "prev_action",
          "joint_nominal", "joint_default", "done"]
TERMS = ["lin_vel_tracking", "ang_vel_tracking", "feet_airtime", "feet_clearance", "feet_phase",
         "feet_slip", "orientation", "joint_torque", "joint_position", "action_rate", "energy",
         "pose", "termination", "standstill", "lin_vel_z", "ang_vel_xy"]


def _import():
    sys.path.insert(0, REF)
    from deskrl import envkit, gaitgen, mathcore, randomization, rewards

    return envkit, gaitgen, mathcore, randomization, rewards


def stack_frames(frames):
    out = {}
    for f in FIELDS:
        vals = [getattr(fr, f) for fr in frames]
        if f in ("foot_contact", "touchdown"):
            out[f] = np.array(vals, dtype=np.uint8)
        elif f == "done":
            out[f] = np.array([bool(v) for v in vals], dtype=np.uint8)
        else:
            out[f] = np.array(vals, dtype=np.float64)
    return out


def frames_case(gaitgen, rng, nj, nf, n_random, n_gait):
    frames = [gaitgen.random_frame(rng, nj, nf) for _ in range(n_random)]
    gen = gaitgen.GaitGenerator(gaitgen.GaitGeneratorConfig(num_joints=nj, num_feet=nf), seed=3)
    frames += [gen.step() for _ in range(n_gait)]
    # edge cases: zero command (standstill gate), exactly-zero foot speed
    f0 = gaitgen.random_frame(rng, nj, nf)
    f0.command = np.array([0.05, -0.02, 0.3])
    f0.foot_vel_xy = np.zeros((nf, 2))
    frames.append(f0)
    return frames


def main():
    envkit, gaitgen, mathcore, randomization, rewards = _import()
    data = {}
    rng = np.random.default_rng(11)
    cfgs = {
        "default": rewards.RewardTermConfig(),
        "gated": rewards.RewardTermConfig(standstill_gated=True, w_lin_vel=1.5, sigma_phase=0.01,
                                          w_energy=-2e-3, airtime_min=0.05, airtime_max=0.4),
    }
    noise = envkit.ObservationNoise(gravity=0.05, lin_vel=0.1, ang_vel=0.2, joint_pos=0.01,
                                    joint_vel=1.5)
    partial_noise = envkit.ObservationNoise(gravity=0.0, lin_vel=0.1, ang_vel=0.0, joint_pos=0.03,
                                            joint_vel=0.0)
    for shape, (nj, nf) in {"go1": (12, 4), "biped": (8, 2)}.items():
        frames = frames_case(gaitgen, rng, nj, nf, 192, 64)
        n = len(frames)
        for k, v in stack_frames(frames).items():
            data[f"{shape}/frame/{k}"] = v
        for cname, cfg in cfgs.items():
            terms = np.zeros((n, len(TERMS)))
            unclipped = np.zeros(n)
            total = np.zeros(n)
            for i, fr in enumerate(frames):
                b = rewards.total_reward(fr, cfg)
                terms[i] = [b.terms[t] for t in TERMS]
                unclipped[i] = b.unclipped_total
                total[i] = b.total
            data[f"{shape}/reward/{cname}/terms"] = terms
            data[f"{shape}/reward/{cname}/unclipped"] = unclipped
            data[f"{shape}/reward/{cname}/total"] = total
        # observations: noise streams keyed like the env (seed, env, episode, step)
        pert = rng.normal(0, 3, (n, 3))
        for oname, nz in {"noisy": noise, "partial": partial_noise, "clean": None}.items():
            st, pr = [], []
            for i, fr in enumerate(frames):
                g = envkit.stream_rng(77, 1000 + i, 2, 5) if nz is not None else None
                o = envkit.build_locomotion_observation(fr, fr.prev_action, fr.command, nz, g,
                                                        pert[i] if oname != "clean" else None)
                st.append(o["state"])
                pr.append(o["privileged_state"])
            data[f"{shape}/obs/{oname}/state"] = np.array(st)
            data[f"{shape}/obs/{oname}/priv"] = np.array(pr)
        data[f"{shape}/obs/pert"] = pert
    data["obs/noise"] = np.array([noise.gravity, noise.lin_vel, noise.ang_vel, noise.joint_pos,
                                  noise.joint_vel])
    data["obs/partial_noise"] = np.array([partial_noise.gravity, partial_noise.lin_vel,
                                          partial_noise.ang_vel, partial_noise.joint_pos,
                                          partial_noise.joint_vel])
    data["obs/key"] = np.array([77, 1000, 2, 5], dtype=np.int64)  # seed, env0, episode, step

    # project_gravity KATs (+ non-unit rejection)
    qs = np.array([mathcore.sample_uniform_quaternion(rng) for _ in range(256)])
    data["gravity/q"] = qs
    data["gravity/out"] = np.array([mathcore.project_gravity(q) for q in qs])
    bad = qs[:4] * np.array([1.0 + 2e-6, 1.0 - 3e-6, 1.0 + 5e-7, 1.0])[:, None]
    ok = []
    for q in bad:
        try:
            mathcore.project_gravity(q)
            ok.append(1)
        except mathcore.InvalidInputError:
            ok.append(0)
    data["gravity/bad_q"] = bad
    data["gravity/bad_ok"] = np.array(ok, dtype=np.uint8)

    # phase
    phi = rng.uniform(-math.pi, math.pi, (128, 4))
    phi[0] = [-math.pi, math.pi - 1e-12, 0.0, 3.0]
    freqs = rng.uniform(0.5, 3.0, 128)
    dts = rng.choice([0.01, 0.02, 0.004], 128)
    adv = []
    for i in range(128):
        ps = mathcore.PhaseState(phi=np.clip(phi[i], -math.pi, np.nextafter(math.pi, 0)),
                                 frequency=float(freqs[i]), dt=float(dts[i]))
        adv.append(mathcore.advance_phase(ps).phi)
    data["phase/phi"] = np.clip(phi, -math.pi, np.nextafter(math.pi, 0))
    data["phase/freq"] = freqs
    data["phase/dt"] = dts
    data["phase/advanced"] = np.array(adv)
    data["phase/encoded"] = mathcore.phase_encode(data["phase/phi"])
    wr = rng.uniform(-40, 40, 512)
    data["phase/wrap_in"] = wr
    data["phase/wrap_out"] = mathcore.wrap_angle(wr)
    data["phase/swing"] = rewards.swing_height_profile(data["phase/phi"], 0.08)

    # PD mapping
    J = 12
    qdef = rng.normal(0, 0.3, J)
    a = rng.uniform(-1.5, 1.5, (64, J))
    prev = rng.normal(0, 0.5, (64, J))
    q = rng.normal(0, 0.5, (64, J))
    v = rng.normal(0, 2.0, (64, J))
    pabs = envkit.PDParams(kp=35.0, kd=0.5, action_scale=0.3, q_default=qdef, torque_limit=20.0)
    prel = envkit.PDParams(kp=20.0, kd=1.0, action_scale=0.25, q_default=qdef, mode="relative",
                           torque_limit=np.inf, joint_range=(-0.8, 0.9))
    data["pd/qdef"], data["pd/a"], data["pd/prev"], data["pd/q"], data["pd/v"] = qdef, a, prev, q, v
    for name, pp in (("abs", pabs), ("rel", prel)):
        tgt = np.array([envkit.action_to_target(a[i], prev[i], pp) for i in range(64)])
        tau = np.array([envkit.pd_torque(tgt[i], q[i], v[i], pp) for i in range(64)])
        data[f"pd/{name}/target"] = tgt
        data[f"pd/{name}/torque"] = tau
        data[f"pd/{name}/params"] = np.array([pp.kp, pp.kd, pp.action_scale, pp.torque_limit,
                                              pp.joint_range[0], pp.joint_range[1],
                                              1.0 if pp.mode == "relative" else 0.0])

    # progress clip
    raw = rng.normal(0, 1, 256)
    hist = np.where(rng.uniform(size=256) < 0.2, 0.0, rng.normal(0, 1, 256))
    pc = np.array([envkit.progress_clip_reward(float(r), float(h)) for r, h in zip(raw, hist)])
    data["progress/raw"], data["progress/hist"], data["progress/out"] = raw, hist, pc

    # sensor noise (uniform) and pose injection, Philox-keyed streams
    obs = rng.normal(0, 1, (32, 9))
    specs = (randomization.NoiseSpec("a", 0.1), randomization.NoiseSpec("b", 0.0),
             randomization.NoiseSpec("c", 0.5))
    noised = []
    for i in range(32):
        d = {"a": obs[i, :3], "b": obs[i, 3:6], "c": obs[i, 6:]}
        o = randomization.apply_sensor_noise(d, specs, envkit.stream_rng(5, i, 0, 1))
        noised.append(np.concatenate([o["a"], o["b"], o["c"]]))
    data["dr/noise_in"], data["dr/noise_out"] = obs, np.array(noised)
    pose = rng.normal(0, 1, (64, 7))
    bounds = np.stack([np.full(7, -0.5), np.linspace(0.1, 1.0, 7)], axis=1)
    inj = np.array([randomization.pose_injection(pose[i], envkit.stream_rng(9, i, 3, 0), 0.4,
                                                 bounds) for i in range(64)])
    data["dr/pose_in"], data["dr/pose_bounds"], data["dr/pose_out"] = pose, bounds, inj

    # gaussian + uniform sensor noise (randomization.py:103-106, Generator.normal)
    obs_g = rng.normal(0, 1, (48, 10))
    specs_g = (randomization.NoiseSpec("a", 0.2, "gaussian"), randomization.NoiseSpec("b", 0.05),
               randomization.NoiseSpec("c", 1.5, "gaussian"))
    noised = []
    for i in range(48):
        d = {"a": obs_g[i, :4], "b": obs_g[i, 4:6], "c": obs_g[i, 6:]}
        o = randomization.apply_sensor_noise(d, specs_g, envkit.stream_rng(6, 100 + i, 1, 7))
        noised.append(np.concatenate([o["a"], o["b"], o["c"]]))
    data["dr/gnoise_in"], data["dr/gnoise_out"] = obs_g, np.array(noised)

    # known answers of one stream: Generator.standard_normal / integers
    data["dr/normal_known"] = envkit.stream_rng(0, 0, 0, 0).standard_normal(4096)
    g = envkit.stream_rng(0, 0, 0, 0)
    data["dr/int_known"] = np.array([int(g.integers(1, 4)) for _ in range(64)])

    # randomize_params on DynamicsParams (randomization.py:156-181): additive with
    # resampling (pole_mass 0.1 + U(-0.3, 0.2) is often non-positive), multiplicative,
    # log-uniform, and an additive range on a zero field (link_damping: no check)
    from deskrl import dynamics
    nominal = dynamics.DynamicsParams()
    pnames = [f.name for f in dataclasses.fields(nominal)]
    ranges = (randomization.ParamRange("pole_mass", "uniform_additive", -0.3, 0.2),
              randomization.ParamRange("cart_mass", "uniform_multiplicative", 0.5, 1.5),
              randomization.ParamRange("pend_damping", "log_uniform", 0.1, 10.0),
              randomization.ParamRange("link_damping", "uniform_additive", -0.1, 0.1),
              randomization.ParamRange("gravity", "uniform_additive", -0.5, 0.5))
    spec = randomization.RandomizationSpec(params=ranges)
    rp = []
    for i in range(64):
        pp = randomization.randomize_params(nominal, spec, envkit.stream_rng(21, i, 4, 0))
        rp.append([getattr(pp, k) for k in pnames])
    data["dr/params_nominal"] = np.array([getattr(nominal, k) for k in pnames])
    data["dr/params_fields"] = np.array(pnames)
    data["dr/params_ranges"] = np.array([[pnames.index(r.path), ("uniform_additive",
                                          "uniform_multiplicative", "log_uniform").index(
                                              r.distribution), r.low, r.high] for r in ranges])
    data["dr/params_out"] = np.array(rp)

    # DelayLine: per-episode (1..3) and per-step (0..5) delays over 24 pushes
    vals = rng.normal(0, 1, (24, 16, 3))
    for mode, (lo, hi, per_step) in (("ep", (1, 3, False)), ("st", (0, 5, True))):
        lines = [randomization.DelayLine(lo, hi, per_step) for _ in range(16)]
        for i, ln in enumerate(lines):
            ln.reset(envkit.stream_rng(31, i, 2, 0))
        outs = []
        for t in range(24):
            outs.append([np.asarray(ln.push_pop(vals[t, i], envkit.stream_rng(32, i, 2, t)))
                         for i, ln in enumerate(lines)])
        data[f"dr/delay_{mode}_out"] = np.array(outs)
        data[f"dr/delay_{mode}_delay"] = np.array([ln._episode_delay for ln in lines])
    data["dr/delay_in"] = vals

    # curriculum: a success sequence per learner
    seq = rng.uniform(size=(16, 40)) < 0.6
    lv = []
    for s in seq:
        c = randomization.CurriculumState(promotion_threshold=2, max_level=5)
        hist_c = []
        for x in s:
            c = randomization.curriculum_update(c, bool(x))
            hist_c.append([c.level, c.successes_at_level, c.episodes, c.total_successes])
        lv.append(hist_c)
    data["dr/curr_seq"] = seq.astype(np.uint8)
    data["dr/curr_out"] = np.array(lv, dtype=np.int64)

    data["terms"] = np.array(TERMS)
    data["fields"] = np.array(FIELDS)
    path = os.path.join(OUT, "loco_golden.npz")
    np.savez_compressed(path, **data)
    print(f"wrote {path} ({os.path.getsize(path)} bytes, {len(data)} arrays)")


if __name__ == "__main__":
    main()
