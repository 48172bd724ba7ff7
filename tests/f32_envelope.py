"""float32 tolerance floors derived from f32 rounding (BASELINE.md
"Parity").

The BASELINE tolerance for the float32 build is 1e-5 relative after 1 step
and 1e-3 over 100 steps, relative to max(|ref|, floor).  With a single 1e-3
floor some components fail in EVERY float32 implementation, the correctly
rounded restatement included (build DK_F32_FAITHFUL, profiles/r02_f32_ab.json):
the sine of a pendulum angle near pi, reacher's target - tip (operands of size
~2 subtracted), and cartpole's angular velocity after 100 chaotic steps.  The
floor of each observation component is therefore derived from the rounding
itself: E_c(h) is the largest deviation, over every world and step <= h, of
the float64 oracle run with its state (and observation) rounded to float32
after every step -- the error storage in float32 alone produces, before any
float32 arithmetic -- and

    floor_c(h) = max(1e-3, K * E_c(h) / rtol(h)),  K = 4,

so a component whose reference value is small may deviate by at most K times
what rounding the state to float32 already causes.  Computed by the CPU oracle
on the test's own inputs; nothing here touches the GPU.
"""

import numpy as np

K_ULP = 4.0
RTOL_1, RTOL_H = 1e-5, 1e-3


def r32(x):
    return np.asarray(x, np.float64).astype(np.float32).astype(np.float64)


def envelope(oracle, task, n, seed, acts, mid_reset_step=-1, round_actions=True, **kw):
    """(ref_obs [K, n, O], E [K, O]): E[k] = max deviation over worlds and steps
    <= k of the float32-state oracle (actions rounded to float32 too, as the
    float32 kernel receives them) from the exact one."""
    emu_acts = r32(acts) if round_actions else acts
    ref = oracle.OracleBatchEnv(task, n, **kw)
    emu = oracle.OracleBatchEnv(task, n, **kw)
    ref.reset(seed=seed)
    emu.reset(seed=seed)
    emu.state[:] = r32(emu.state)
    emu.target[:] = r32(emu.target)
    obs, E = [], []
    run = None
    for k in range(acts.shape[0]):
        if k == mid_reset_step:
            ref.reset()
            emu.reset()
            emu.state[:] = r32(emu.state)
            emu.target[:] = r32(emu.target)
        o_r = ref.step(acts[k])[0]
        o_e = emu.step(emu_acts[k])[0]
        emu.state[:] = r32(emu.state)
        d = np.abs(r32(o_e) - o_r).max(axis=0)
        run = d if run is None else np.maximum(run, d)
        obs.append(o_r)
        E.append(run.copy())
    return np.stack(obs), np.stack(E)


def reset_envelope(oracle, task, n, seed, resets=2, **kw):
    """E_c of the reset observation: the float32-rounded reset state's
    observation (rounded) against the exact one, per component, over the
    first `resets` episodes' draws."""
    env = oracle.OracleBatchEnv(task, n, **kw)
    params = kw.get("params")
    E = None
    for k in range(resets):
        obs0 = env.reset(seed=seed) if k == 0 else env.reset()
        E = np.zeros(obs0.shape[1]) if E is None else E
        for w in range(n):
            o = oracle.state_obs(task, r32(env.state[w]), r32(env.target[w]), params)
            E = np.maximum(E, np.abs(r32(o) - obs0[w]))
    return E


def floors(E_k, rtol):
    return np.maximum(1e-3, K_ULP * np.asarray(E_k) / rtol)


def rel_err(got, want, floor):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    return float((np.abs(got - want) / np.maximum(np.abs(want), floor)).max())
