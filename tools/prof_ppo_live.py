"""Per-kernel device time of the PPO rollout phase as it runs (CUDA-graph
replay, no serialisation): torch.profiler's CUPTI activity over a few
RolloutGraph phases.  python tools/prof_ppo_live.py [--go1]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from torch.profiler import ProfilerActivity, profile

    import paper_2502_08844_b200 as dk
    from paper_2502_08844_b200 import ppo as P
    from paper_2502_08844_b200 import rollout as R

    class Cfg:
        unroll_length, reward_scaling, discounting = 30, 10.0, 0.995
        policy_obs_key = value_obs_key = "state"

    torch.manual_seed(0)
    n = 8192
    if "--go1" in sys.argv:  # the Go1 joystick env, asymmetric actor-critic
        from paper_2502_08844_b200 import go1env as G
        Cfg.value_obs_key = "privileged_state"
        env = G.DeviceGo1Env(n, G.Go1Config(), dtype="float32")
        dp, dv, na = 56, 75, 12
    else:
        env = dk.DeviceBatchEnv(dk.EnvConfig(task="cartpole-balance"), n, dtype="float32")
        dp, dv, na = 5, 5, 1
    obs = env.reset(seed=0)
    policy, value = R.make_policy(dp, na).cuda(), R.make_value(dv).cuda()
    rg = R.RolloutGraph(env, policy, value, Cfg, obs, P.DeviceRunningNormalizer(dp),
                        P.DeviceRunningNormalizer(dv))
    for _ in range(3):
        rg.run()
    torch.cuda.synchronize()
    phases = 4
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(phases):
            rg.run()
        torch.cuda.synchronize()
    rows = {}
    for e in prof.events():
        if e.device_type.name != "CUDA":
            continue
        k = e.name[:90]
        t, c = rows.get(k, (0.0, 0))
        rows[k] = (t + e.device_time, c + 1)
    tot = sum(t for t, _ in rows.values())
    print(f"total device time per phase {tot / phases / 1e3:.3f} ms "
          f"({tot / phases / Cfg.unroll_length:.1f} us per step)")
    for k, (t, c) in sorted(rows.items(), key=lambda kv: -kv[1][0])[:30]:
        print(f"{t / phases:9.1f} us/phase {100 * t / tot:5.1f}% {c // phases:4d}/phase  {k}")


if __name__ == "__main__":
    main()
