"""On-device PPO rollout collection (ppo.py:295-378).

``collect_rollout_device`` is ``ppo.collect_rollout`` with every tensor kept on
the GPU: the policy and value networks (the reference's own ``torch.nn``
modules, moved to CUDA; their GEMMs are cuBLAS), the env step
(``DeviceBatchEnv.step``, one ``rollout_kernel`` launch per control step), the
running observation normalisers (``DeviceRunningNormalizer``), the truncation
bootstrap through the terminal observation, and the reward scaling.  No
per-step host synchronisation: the terminal-value bootstrap is evaluated for
all worlds every step and masked (the reference evaluates the truncated rows
only after a host-side ``trunc.any()``).

Semantics follow the reference line by line (ppo.py:308-378): observations are
normalised with the pre-phase statistics and stored as the networks saw them;
the raw observations are folded into the normalisers only after the phase;
``rewards = reward * reward_scaling + discounting * terminal_value``;
``dones = done | trunc``.  Sampling noise: ``noise`` [T, N, A] (e.g. the
reference's CPU ``torch.randn`` draws, for parity tests) or a CUDA generator.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

from . import _native as nat
from .envkit import ConfigError, _check


@dataclass
class DeviceRolloutBatch:
    """ppo.RolloutBatch (ppo.py:245-256) with CUDA tensors [T, N, ...]."""

    policy_obs: object
    value_obs: object
    actions: object
    pre_tanh: object
    log_probs: object
    rewards: object
    dones: object
    values: object
    bootstrap: object
    raw_policy_obs: object = None  # [T*N, O] raw observations of the phase (normaliser input)
    raw_value_obs: object = None
    nan_flag: object = None  # device bool: the policy produced a NaN mean in this phase


_LOG_2 = 0.6931471805599453


def _mlp(sizes, out_dim):
    import torch.nn as nn

    layers = []
    for a, b in zip(sizes[:-1], sizes[1:]):
        layers += [nn.Linear(a, b), nn.SiLU()]
    layers.append(nn.Linear(sizes[-1], out_dim))
    return nn.Sequential(*layers)


def make_policy(obs_dim: int, action_dim: int, hidden=(128, 128, 128, 128),
                init_std: float = 0.5):
    """ppo.MLPPolicy (ppo.py:121-133): Linear/Swish trunk + a free log_std;
    forward(obs) -> (mean, log_std).  Same parameter names, so the reference's
    state_dict loads unchanged."""
    import math

    import torch
    import torch.nn as nn

    class MLPPolicy(nn.Module):
        def __init__(self):
            super().__init__()
            self.trunk = _mlp((obs_dim, *hidden), action_dim)
            self.log_std = nn.Parameter(torch.full((action_dim,), math.log(init_std)))
            self.action_dim = action_dim

        def forward(self, obs):
            mean = self.trunk(obs)
            return mean, self.log_std.expand_as(mean)

    return MLPPolicy()


def make_cnn_policy(in_channels: int, image_size: int, action_dim: int, dense=(256, 256),
                    init_std: float = 0.5):
    """ppo.CNNPolicy (ppo.py:143-178): conv trunk 32@8x8/4, 64@4x4/2, 64@3x3/1
    (Swish), dense layers, a linear head and a free log_std; input the
    pixel_normalize'd [N, C, H, W] float32 stack.  Same parameter names as the
    reference (trunk.convs.*, trunk.dense.*, head.*, log_std)."""
    import math

    import torch
    import torch.nn as nn

    class CNNTrunk(nn.Module):
        def __init__(self):
            super().__init__()
            self.convs = nn.Sequential(
                nn.Conv2d(in_channels, 32, 8, stride=4), nn.SiLU(),
                nn.Conv2d(32, 64, 4, stride=2), nn.SiLU(),
                nn.Conv2d(64, 64, 3, stride=1, padding=1), nn.SiLU(),
                nn.Flatten(),
            )
            with torch.no_grad():
                flat = self.convs(torch.zeros(1, in_channels, image_size, image_size)).shape[1]
            layers = []
            sizes = (flat, *dense)
            for a, b in zip(sizes[:-1], sizes[1:]):
                layers += [nn.Linear(a, b), nn.SiLU()]
            self.dense = nn.Sequential(*layers)
            self.out_dim = dense[-1]

        def forward(self, img):
            return self.dense(self.convs(img))

    class CNNPolicy(nn.Module):
        def __init__(self):
            super().__init__()
            self.trunk = CNNTrunk()
            self.head = nn.Linear(self.trunk.out_dim, action_dim)
            self.log_std = nn.Parameter(torch.full((action_dim,), math.log(init_std)))
            self.action_dim = action_dim

        def forward(self, img):
            mean = self.head(self.trunk(img))
            return mean, self.log_std.expand_as(mean)

    return CNNPolicy()


def make_value(obs_dim: int, hidden=(256, 256, 256, 256, 256)):
    """ppo.MLPValue (ppo.py:136-142): forward(obs) -> [N] values."""
    import torch.nn as nn

    class MLPValue(nn.Module):
        def __init__(self):
            super().__init__()
            self.trunk = _mlp((obs_dim, *hidden), 1)

        def forward(self, obs):
            return self.trunk(obs).squeeze(-1)

    return MLPValue()


def tanh_gaussian_log_prob(mean, log_std, pre_tanh):
    """ppo.tanh_gaussian_log_prob (the same torch expression, on device)."""
    import math

    import torch

    std = torch.exp(log_std)
    base = -0.5 * (((pre_tanh - mean) / std) ** 2) - log_std - 0.5 * math.log(2 * math.pi)
    correction = 2.0 * (_LOG_2 - pre_tanh - torch.nn.functional.softplus(-2.0 * pre_tanh))
    return (base - correction).sum(-1)


def _sample(mean, log_std, eps, nan_flag, out=None):
    """policy_forward's sampling + tanh_gaussian_log_prob (ppo.py:204-217): one
    fused kernel (dk_ppo_sample) for float32 networks, else the torch
    expressions; NaN means set nan_flag.  out: optional (pre_tanh, action,
    log_prob) float32 buffers to write."""
    import torch

    if (mean.dtype == torch.float32 and eps.dtype == torch.float32 and mean.dim() == 2
            and log_std.dtype == torch.float32 and log_std.stride(-1) == 1):
        m, e = mean.contiguous(), eps.contiguous()
        n, A = m.shape
        if out is not None:
            pre, act, lp = out
        else:
            pre, act = torch.empty_like(m), torch.empty_like(m)
            lp = torch.empty((n,), dtype=torch.float32, device=m.device)
        _check(nat.lib().dk_ppo_sample(n, A, m.data_ptr(), log_std.data_ptr(), log_std.stride(0),
                                       e.data_ptr(), pre.data_ptr(), act.data_ptr(),
                                       lp.data_ptr(), nan_flag.data_ptr(),
                                       torch.cuda.current_stream(m.device).cuda_stream))
        return pre, act, lp
    nan_flag |= torch.isnan(mean).any().to(nan_flag.dtype)
    pre_tanh = mean + torch.exp(log_std) * eps
    res = pre_tanh, torch.tanh(pre_tanh), tanh_gaussian_log_prob(mean, log_std, pre_tanh)
    if out is not None:
        for o, r in zip(out, res):
            o.copy_(r)
        return out
    return res


def _route(obs: dict, cfg):
    for key in (cfg.policy_obs_key, cfg.value_obs_key):
        if key not in obs:
            raise ConfigError(f"observation slot {key!r} missing")
    return obs[cfg.policy_obs_key], obs[cfg.value_obs_key]


def collect_rollout_device(env, policy, value, cfg, obs: dict, policy_normalizer=None,
                           value_normalizer=None, noise=None, generator=None,
                           update_normalizers: bool = True, tensor_cores: bool = True,
                           _op_by_op: bool = False):
    """Unroll ``cfg.unroll_length`` control steps across the batch on the GPU.

    env: DeviceBatchEnv; policy / value: CUDA ``nn.Module``s with the
    reference's MLPPolicy / MLPValue interfaces; obs: the device observation
    dict to resume from; normalisers: DeviceRunningNormalizer or None.
    Returns (DeviceRolloutBatch, next obs dict, mean raw reward tensor).
    """
    import torch

    T, N = int(cfg.unroll_length), env.num_envs
    if tensor_cores:  # the reference-shaped MLPs on tcgen05 (mlp.py); others unchanged
        from .mlp import tc_policy, tc_value

        policy, value = tc_policy(policy), tc_value(value)
    if noise is not None and tuple(noise.shape[:2]) != (T, N):
        raise ConfigError("noise must be [unroll_length, num_envs, action_dim]")
    # ppo.policy_forward's NaN check (ppo.py:208), as a device flag read once
    # per phase instead of one host sync per step
    nan_flag = torch.zeros((), dtype=torch.int32, device=env.device)
    out = env._outputs((), False)  # reused step buffers (stream-ordered)
    f32 = torch.float32
    p_obs, v_obs, acts, pres, lps, rews, dns, vals = [], [], [], [], [], [], [], []
    raw_p, raw_v = [], []
    raw_reward_sum = torch.zeros((), dtype=torch.float64, device=env.device)

    pixel_policy = cfg.policy_obs_key == "pixels"
    if pixel_policy:
        from .pixels import pixel_normalize

    def prep(normalizer, x):
        return (normalizer.apply(x) if normalizer is not None else x).to(f32)

    def prep_policy(x):  # ppo._prep_policy_obs (ppo.py:278-285)
        if pixel_policy:  # NCHW view of an NHWC (channels_last) tensor: 2x faster cuDNN convs
            return pixel_normalize(x, channels_first=False).permute(0, 3, 1, 2)
        return prep(policy_normalizer, x)

    if not (pixel_policy or _op_by_op) and _fused_ok(env, obs, cfg, policy_normalizer,
                                                     value_normalizer):
        return _collect_fused(env, policy, value, cfg, obs, policy_normalizer, value_normalizer,
                              noise, generator, update_normalizers, nan_flag, out)

    with torch.no_grad():
        for t in range(T):
            pol_in, val_in = _route(obs, cfg)
            pol_t, val_t = prep_policy(pol_in), prep(value_normalizer, val_in)
            if policy_normalizer is not None and not pixel_policy:
                raw_p.append(pol_in.clone())
            if value_normalizer is not None:
                raw_v.append(val_in.clone())
            mean, log_std = policy(pol_t)
            eps = noise[t].to(mean.dtype) if noise is not None else torch.randn(
                mean.shape, generator=generator, device=mean.device, dtype=mean.dtype)
            pre_tanh, action, log_prob = _sample(mean, log_std, eps, nan_flag)
            step = env.step(action.to(env.dtype), autoreset=True, with_info=False, out=out)
            reward = step["reward"].to(torch.float64)
            raw_reward_sum += reward.mean()
            # truncation bootstraps through the terminal observation (ppo.py:327-341),
            # for every world at once, masked to the truncated, non-terminated ones
            boot = step["trunc"].bool() & ~step["done"].bool() & step["terminal_mask"].bool()
            term_in = torch.where(boot[:, None], step[_terminal_key(step, cfg)],
                                  torch.zeros((), dtype=env.dtype, device=env.device))
            # the value of the observation and of the terminal observation in one
            # network call (rows are independent): 2N rows fill twice the SMs
            vv = value(torch.cat([val_t, prep(value_normalizer, term_in)]))
            v, tv = vv[:N], vv[N:].to(torch.float64)
            term_val = torch.where(boot, tv, torch.zeros_like(tv))
            p_obs.append(pol_t)
            v_obs.append(val_t)
            acts.append(action.to(torch.float64))
            pres.append(pre_tanh)
            lps.append(log_prob)
            rews.append(reward * cfg.reward_scaling + cfg.discounting * term_val)
            dns.append((step["done"] | step["trunc"]).to(torch.float64))
            vals.append(v.to(torch.float64))
            obs = _next_obs(step, clone=True)
            if "pixels" in step:
                obs["pixels"] = step["pixels"].clone()
        _, val_in = _route(obs, cfg)
        bootstrap = value(prep(value_normalizer, val_in)).to(torch.float64)
    batch = DeviceRolloutBatch(torch.stack(p_obs), torch.stack(v_obs), torch.stack(acts),
                               torch.stack(pres), torch.stack(lps), torch.stack(rews),
                               torch.stack(dns), torch.stack(vals), bootstrap)
    batch.raw_policy_obs = torch.cat(raw_p, 0) if raw_p else None
    batch.raw_value_obs = torch.cat(raw_v, 0) if raw_v else None
    batch.nan_flag = nan_flag
    if not torch.cuda.is_current_stream_capturing():
        _check_phase(env, batch)
    # fold the phase's raw observations into the statistics afterwards (ppo.py:370-377)
    if update_normalizers:
        _update(batch, policy_normalizer, value_normalizer)
    return batch, obs, raw_reward_sum / T


def _next_obs(step, clone=False):
    """The step's observation dict: the policy's ``state`` and the critic's
    ``privileged_state`` (the same tensor for the analytic tasks; the Go1 env
    returns both)."""
    s = step["obs"]
    p = step.get("privileged_state")
    p = s if p is None else p
    if clone:
        s = s.clone()
        p = s if p is step["obs"] else p.clone()
    return {"state": s, "privileged_state": p}


def _terminal_key(step, cfg):
    """The terminal rows the critic bootstraps from: the privileged ones when the
    value network reads ``privileged_state`` and the env returns them."""
    if cfg.value_obs_key == "privileged_state" and step.get("terminal_privileged_state") is not None:
        return "terminal_privileged_state"
    return "terminal_obs"


def _fused_ok(env, obs, cfg, pn, vn):
    """The fused bookkeeping path (dk_ppo_step_*) takes float32 state
    observations and device normalisers (or none)."""
    import torch

    from .ppo import DeviceRunningNormalizer

    if env.dtype != torch.float32:
        return False
    for key in (cfg.policy_obs_key, cfg.value_obs_key):
        x = obs.get(key)
        if x is None or x.dtype != torch.float32 or x.dim() != 2:
            return False
    return all(n is None or isinstance(n, DeviceRunningNormalizer) for n in (pn, vn))


def _norm_c(normalizer):
    if normalizer is None:
        return nat.PpoNormC(None, None, 0.0, 0, 0)
    return nat.PpoNormC(normalizer.mean.data_ptr(), normalizer.var.data_ptr(),
                        float(normalizer.epsilon), int(normalizer.count == 0.0), 1)


def _collect_fused(env, policy, value, cfg, obs, pn, vn, noise, generator, update_normalizers,
                   nan_flag, out):
    """collect_rollout_device with the per-step bookkeeping in three kernels
    (dk_ppo_step_inputs / _bootstrap / _record) writing straight into the
    phase's [T, N, ...] batch buffers: eight launches per control step (inputs,
    policy, noise, sampling, env step, bootstrap, terminal value, record)
    instead of ~30.  With the tensor-core networks the step values of the whole
    phase (and the bootstrap values) are one launch after it, and so are the
    terminal values of the truncated worlds (one count-limited launch and
    dk_ppo_boot_fixup), and the bootstrap, record and next step's inputs are one
    kernel (dk_ppo_step_post): five launches per step.  Same values as the op-by-op path
    (tests/test_gpu_rollout.py)."""
    import torch

    T, N = int(cfg.unroll_length), env.num_envs
    dev = env.device
    lib = nat.lib()
    st = lambda: torch.cuda.current_stream(dev).cuda_stream  # noqa: E731
    f32, f64 = torch.float32, torch.float64
    pol_in, val_in = _route(obs, cfg)
    dp, dv, A = pol_in.shape[1], val_in.shape[1], env.action_dim
    e = lambda *s_, d=f32: torch.empty(s_, dtype=d, device=dev)  # noqa: E731
    p_obs = e(T, N, dp)
    raw_p = e(T, N, dp) if pn is not None else None
    raw_v = e(T, N, dv) if vn is not None else None
    acts, pres, lps = e(T, N, A, d=f64), e(T, N, A), e(T, N)
    rews, dns, vals = e(T, N, d=f64), e(T, N, d=f64), e(T, N, d=f64)
    value_count = getattr(value, "call_count", None)
    from .mlp import _TCPolicy, _TCValue

    pair = isinstance(policy, _TCPolicy) and isinstance(value, _TCValue)
    # the per-step value call's rows (this step's normalised inputs); with the
    # tensor-core nets the values are evaluated after the phase from v_obs
    vin = None if pair else e(N, dv)
    # the boot rows' terminal observations, compacted (count on the device): per
    # step; or, with the tensor-core nets, over the whole phase into one value
    # input buffer -- rows [0, T N) the step inputs (the batch's value_obs),
    # [T N, T N + N) the final observations' (bootstrap), then the terminal rows
    # (slots counted from T N + N): one count-limited value call after the phase
    # and dk_ppo_boot_fixup
    if pair:
        vbuf = e((2 * T + 1) * N, dv)
        v_obs = vbuf[:T * N].view(T, N, dv)
        vterm = vbuf
        count = torch.full((1,), T * N + N, dtype=torch.int64, device=dev)
    else:
        v_obs = e(T, N, dv)
        vterm = torch.zeros((N, dv), dtype=f32, device=dev)
        count = torch.zeros((1,), dtype=torch.int64, device=dev)
    pos = torch.empty((T, N) if pair else (1, N), dtype=torch.int32, device=dev)
    act = e(N, A)
    nb = int(lib.dk_ppo_record_blocks(N))
    partial = e(T, nb, d=f64)
    np_c, nv_c = _norm_c(pn), _norm_c(vn)
    ptr = lambda x: None if x is None else x.data_ptr()  # noqa: E731
    with torch.no_grad():
        def inputs(t, o):  # dk_ppo_step_inputs: step t's normalised inputs from obs o
            pol_in, val_in = _route(o, cfg)
            pol_in, val_in = pol_in.contiguous(), val_in.contiguous()
            _check(lib.dk_ppo_step_inputs(
                N, dp, dv, pol_in.data_ptr(), val_in.data_ptr(), ctypes.byref(np_c),
                ctypes.byref(nv_c), ptr(None if raw_p is None else raw_p[t]),
                ptr(None if raw_v is None else raw_v[t]), p_obs[t].data_ptr(), v_obs[t].data_ptr(),
                ptr(vin), st()))

        if pair and T > 0:
            inputs(0, obs)
        for t in range(T):
            if not pair:
                inputs(t, obs)
            # (pair: the value of this step's inputs is evaluated with the whole
            # phase's after it, in one launch: rows are independent, the
            # normaliser is constant within the phase, so the values are the same)
            mean, log_std = policy(p_obs[t])
            eps = noise[t].to(mean.dtype) if noise is not None else torch.randn(
                mean.shape, generator=generator, device=mean.device, dtype=mean.dtype)
            _sample(mean, log_std, eps, nan_flag, out=(pres[t], act, lps[t]))
            step = env.step(act, autoreset=True, with_info=False, out=out)
            if pair:
                # bootstrap + record of this step and the next step's inputs: one launch
                nxt = None
                if t + 1 < T:
                    np_in, nv_in = _route(_next_obs(step), cfg)
                    if np_in.is_contiguous() and nv_in.is_contiguous():
                        nxt = (np_in, nv_in)
                post = nat.PpoPostC(
                    n=N, dp=dp, dv=dv, action_dim=A, done=step["done"].data_ptr(),
                    trunc=step["trunc"].data_ptr(), terminal_mask=step["terminal_mask"].data_ptr(),
                    terminal_obs=step[_terminal_key(step, cfg)].data_ptr(),
                    val_term=vterm.data_ptr(), count=count.data_ptr(), pos=pos[t].data_ptr(),
                    dones=dns[t].data_ptr(), reward=step["reward"].data_ptr(),
                    action=act.data_ptr(), reward_scaling=float(cfg.reward_scaling),
                    discounting=float(cfg.discounting), rewards_out=rews[t].data_ptr(),
                    actions_out=acts[t].data_ptr(), reward_partial=partial[t].data_ptr(),
                    next_obs_p=ptr(nxt[0]) if nxt else None,
                    next_obs_v=ptr(nxt[1]) if nxt else None,
                    next_raw_p=ptr(raw_p[t + 1]) if nxt and raw_p is not None else None,
                    next_raw_v=ptr(raw_v[t + 1]) if nxt and raw_v is not None else None,
                    next_pol=ptr(p_obs[t + 1]) if nxt else None,
                    next_val=ptr(v_obs[t + 1]) if nxt else None)
                _check(lib.dk_ppo_step_post(ctypes.byref(post), ctypes.byref(np_c),
                                            ctypes.byref(nv_c), st()))
                if t + 1 < T and nxt is None:  # (strided observations: separately)
                    inputs(t + 1, _next_obs(step))
            else:
                _check(lib.dk_ppo_step_bootstrap(
                    N, dv, step["done"].data_ptr(), step["trunc"].data_ptr(),
                    step["terminal_mask"].data_ptr(), step[_terminal_key(step, cfg)].data_ptr(),
                    ctypes.byref(nv_c), vterm.data_ptr(), count.data_ptr(), pos[0].data_ptr(),
                    dns[t].data_ptr(), st()))
                v = value(vin)
                # terminal values: the compacted boot rows only (tensor-core MLP with a
                # device-side row count), else the whole buffer (rows past the count unread)
                vt = value_count(vterm, count) if value_count is not None else value(vterm)
                v, vt = (x if x.dtype == f32 and x.is_contiguous() else x.to(f32).contiguous()
                         for x in (v, vt))
                _check(lib.dk_ppo_step_record(
                    N, A, step["reward"].data_ptr(), pos[0].data_ptr(), v.data_ptr(),
                    vt.data_ptr(), act.data_ptr(), float(cfg.reward_scaling),
                    float(cfg.discounting), rews[t].data_ptr(), vals[t].data_ptr(),
                    acts[t].data_ptr(), partial[t].data_ptr(), st()))
            # read by the next step's inputs kernel before the env overwrites them
            obs = _next_obs(step)
        if T > 0:
            obs = _next_obs(step, clone=True)  # the phase's last observations, kept
        _, val_in = _route(obs, cfg)
        boot_in = vn.apply(val_in).to(f32) if vn is not None else val_in
        if pair and T > 0:
            # the phase's values, the bootstrap values and the terminal rows' values
            # in one count-limited launch (T N rows fill every SM; per step they
            # were 64 of 148), then the boot rows' reward targets
            vbuf[T * N:T * N + N].copy_(boot_in)
            y = value_count(vbuf, count)
            vals.copy_(y[:T * N].view(T, N))
            bootstrap = y[T * N:T * N + N].to(f64)
            _check(lib.dk_ppo_boot_fixup(T * N, pos.data_ptr(), y.data_ptr(),
                                         float(cfg.discounting), rews.data_ptr(), st()))
        else:
            bootstrap = value(boot_in).to(f64)
    batch = DeviceRolloutBatch(p_obs, v_obs, acts, pres, lps, rews, dns, vals, bootstrap)
    batch.raw_policy_obs = raw_p.reshape(T * N, dp) if raw_p is not None else None
    batch.raw_value_obs = raw_v.reshape(T * N, dv) if raw_v is not None else None
    batch.nan_flag = nan_flag
    if not torch.cuda.is_current_stream_capturing():
        _check_phase(env, batch)
    if update_normalizers:
        _update(batch, pn, vn)
    mean_reward = (partial.sum(1) / N).sum() / T
    return batch, obs, mean_reward


def _check_phase(env, batch):
    """One host sync per phase: the policy's NaN flag (ppo.py:208 raises
    RuntimeError('policy produced NaN mean')) and the env's sticky device
    error word (a rejected step leaves its worlds untouched)."""
    if bool(batch.nan_flag):
        raise RuntimeError("policy produced NaN mean")
    env.check()


def evaluate_device(policy, env, cfg, episodes: int | None = None, max_steps: int | None = None,
                    policy_normalizer=None) -> dict:
    """ppo.evaluate (ppo.py:479-502) on the device: a deterministic-policy
    rollout (action = tanh(mean)), one episode per world, from ``env.reset()``
    until every world has finished once (done | trunc) or ``max_steps`` /
    ``episode_length`` steps.  Returns the reference's dict; stops at exactly
    the reference's step (one 1-byte device→host read per step), so the env's
    episode counters end where the reference's do."""
    import torch

    pixel_policy = cfg.policy_obs_key == "pixels"
    if pixel_policy:
        from .pixels import pixel_normalize
    obs = env.reset()
    n = env.num_envs
    returns = torch.zeros(n, dtype=torch.float64, device=env.device)
    finished = torch.zeros(n, dtype=torch.bool, device=env.device)
    out = env._outputs((), False)
    steps = 0
    limit = max_steps or env.config.episode_length
    with torch.no_grad():
        while steps < limit:
            x = obs[cfg.policy_obs_key]
            if pixel_policy:
                x = pixel_normalize(x, channels_first=False).permute(0, 3, 1, 2)
            else:
                x = (policy_normalizer.apply(x) if policy_normalizer is not None else x)
                x = x.to(torch.float32)
            mean, _ = policy(x)
            if torch.isnan(mean).any():
                raise RuntimeError("policy produced NaN mean")
            step = env.step(torch.tanh(mean).to(env.dtype), autoreset=True, with_info=False,
                            out=out)
            returns += step["reward"].to(torch.float64) * (~finished)
            finished |= step["done"] | step["trunc"]
            steps += 1
            obs = {"state": step["obs"], "privileged_state": step["obs"]}
            if "pixels" in step:
                obs["pixels"] = step["pixels"]
            if bool(finished.all()):
                break
    return {"eval_return_mean": float(returns.mean()),
            "eval_return_std": float(returns.std(unbiased=False)),
            "eval_episode_steps": steps}


def _update(batch, policy_normalizer, value_normalizer):
    if batch.raw_policy_obs is not None:
        policy_normalizer.update(batch.raw_policy_obs)
    if batch.raw_value_obs is not None:
        value_normalizer.update(batch.raw_value_obs)


class RolloutGraph:
    """``collect_rollout_device`` captured once as a CUDA graph and replayed
    per phase: the ~40 small kernels of a control step (two MLPs, sampling,
    env step, bootstrap, bookkeeping) then cost one graph launch per phase
    instead of ~40 Python-dispatched launches per step.  The normaliser
    statistics are device tensors read by the replayed kernels; their update
    (which needs the host-side count) runs eagerly after each replay.  Capture
    happens after a first eager phase, so the normalisers' "count == 0: copy"
    branch is already decided.  Noise comes from torch's default CUDA
    generator (graph-safe Philox offsets)."""

    def __init__(self, env, policy, value, cfg, obs: dict, policy_normalizer=None,
                 value_normalizer=None, tensor_cores: bool = True):
        import torch

        if tensor_cores:
            from .mlp import tc_policy, tc_value

            policy, value = tc_policy(policy), tc_value(value)
        if cfg.policy_obs_key == "pixels":
            raise ConfigError("RolloutGraph: pixel policies run eagerly (collect_rollout_device)")
        self.env, self.policy, self.value, self.cfg = env, policy, value, cfg
        self.pn, self.vn = policy_normalizer, value_normalizer
        # one eager phase: warms up cuBLAS / allocator and fills the statistics
        batch, obs, self.mean_reward = collect_rollout_device(
            env, policy, value, cfg, obs, policy_normalizer, value_normalizer,
            tensor_cores=False)  # (already wrapped above when requested)
        # static observation inputs of the graph: one tensor when the policy and
        # the critic read the same observation, two for an asymmetric critic
        st = obs["state"].clone()
        pv = obs.get("privileged_state")
        pv = st if pv is None or pv is obs["state"] else pv.clone()
        self.obs_in = {"state": st, "privileged_state": pv}
        self.last = batch
        # the capture warm-up really steps the env: snapshot the worlds (state,
        # counters, episode) and the sampling generator, and restore both
        # afterwards so the first replay continues exactly where the eager
        # phase stopped (envs without set_state -- the Go1 env -- advance one
        # extra phase here instead)
        restorable = hasattr(env, "set_state")
        snap = env.state() if restorable else None
        gen_state = torch.cuda.get_rng_state(env.device)
        side = torch.cuda.Stream(device=env.device)
        side.wait_stream(torch.cuda.current_stream(env.device))
        with torch.cuda.stream(side):  # capture warm-up on a side stream
            _, warm_obs, _ = collect_rollout_device(env, policy, value, cfg, dict(self.obs_in),
                                                    policy_normalizer, value_normalizer,
                                                    update_normalizers=False, tensor_cores=False)
        torch.cuda.current_stream(env.device).wait_stream(side)
        torch.cuda.synchronize(env.device)
        if restorable:
            env.set_state(state=snap[0], target=snap[1], steps=snap[2], episode=snap[3],
                          needs_reset=snap[4])
            torch.cuda.set_rng_state(gen_state, env.device)
        else:
            # the env moved on: so does the noise (no phase repeats the warm-up's draws)
            self._copy_obs(warm_obs)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.batch, self.obs_out, self.reward_out = collect_rollout_device(
                env, policy, value, cfg, dict(self.obs_in), policy_normalizer, value_normalizer,
                update_normalizers=False, tensor_cores=False)

    def _copy_obs(self, obs):
        self.obs_in["state"].copy_(obs["state"])
        if self.obs_in["privileged_state"] is not self.obs_in["state"]:
            self.obs_in["privileged_state"].copy_(obs["privileged_state"])

    def run(self, obs: dict | None = None):
        """One phase from ``obs`` (default: where the previous phase stopped).
        Returns (batch, next obs, mean raw reward); the batch tensors are the
        graph's static outputs, overwritten by the next ``run``."""
        if obs is not None and obs["state"].data_ptr() != self.obs_in["state"].data_ptr():
            self._copy_obs(obs)
        self.graph.replay()
        _check_phase(self.env, self.batch)
        _update(self.batch, self.pn, self.vn)
        self._copy_obs(self.obs_out)
        return self.batch, dict(self.obs_in), self.reward_out


__all__ = ["DeviceRolloutBatch", "RolloutGraph", "collect_rollout_device", "evaluate_device",
           "make_cnn_policy",
           "make_policy", "make_value", "tanh_gaussian_log_prob"]
