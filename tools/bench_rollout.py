"""Time collect_rollout_device (policy + value inference + env step + normalisers)
at the reference's default network sizes.  python tools/bench_rollout.py"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2502_08844_b200 as dk
    from paper_2502_08844_b200 import ppo as P
    from paper_2502_08844_b200 import rollout as R

    N = int(os.environ.get("N", 8192))
    T = int(os.environ.get("T", 30))

    class Cfg:
        unroll_length, reward_scaling, discounting = T, 10.0, 0.995
        policy_obs_key = value_obs_key = "state"

    if os.environ.get("TF32"):
        torch.backends.cuda.matmul.allow_tf32 = True
    for dtype in ("float32",):
        env = dk.DeviceBatchEnv(dk.EnvConfig(task="cartpole-balance"), N, dtype=dtype)
        obs = env.reset(seed=0)
        policy = R.make_policy(5, 1).cuda()
        value = R.make_value(5).cuda()
        pn, vn = P.DeviceRunningNormalizer(5), P.DeviceRunningNormalizer(5)
        gen = torch.Generator(device="cuda")
        gen.manual_seed(0)
        for _ in range(3):
            batch, obs, _ = R.collect_rollout_device(env, policy, value, Cfg, obs, pn, vn,
                                                     generator=gen)
        torch.cuda.synchronize()
        reps = 10
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0 = time.perf_counter()
        e0.record()
        for _ in range(reps):
            batch, obs, _ = R.collect_rollout_device(env, policy, value, Cfg, obs, pn, vn,
                                                     generator=gen)
            adv, ret = P.compute_gae_batch(batch.rewards, batch.values, batch.bootstrap,
                                           batch.dones, 0.995, 0.95)
        e1.record()
        torch.cuda.synchronize()
        host = time.perf_counter() - h0
        ms = e0.elapsed_time(e1)
        env.check()
        print(f"collect_rollout_device {dtype}: N={N} T={T}: {reps * T * N / (ms / 1e3):.3e} "
              f"env-steps/s (device {ms / reps:.2f} ms per phase, host {host / reps * 1e3:.2f} ms)")
        rg = R.RolloutGraph(env, policy, value, Cfg, obs, pn, vn)
        for _ in range(3):
            rg.run()
        torch.cuda.synchronize()
        h0 = time.perf_counter()
        e0.record()
        for _ in range(reps):
            batch, obs, _ = rg.run()
            adv, ret = P.compute_gae_batch(batch.rewards, batch.values, batch.bootstrap,
                                           batch.dones, 0.995, 0.95)
        e1.record()
        torch.cuda.synchronize()
        host = time.perf_counter() - h0
        ms = e0.elapsed_time(e1)
        env.check()
        print(f"RolloutGraph {dtype}: N={N} T={T}: {reps * T * N / (ms / 1e3):.3e} "
              f"env-steps/s (device {ms / reps:.2f} ms per phase, host {host / reps * 1e3:.2f} ms)")


if __name__ == "__main__":
    main()
