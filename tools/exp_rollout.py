"""Time fused rollouts (ns per env step) at several world counts -- for A/B of
experimental builds (DK_LIB_PATH=...).  Not a bench line: no roofline/clocks.

    python tools/exp_rollout.py [--dtype float32] [--worlds 4736,8192] [--steps 1000]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--task", default="cartpole-balance")
    ap.add_argument("--dtype", default="float32")
    ap.add_argument("--worlds", default="4736,8192")
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--launches", type=int, default=20)
    ap.add_argument("--tag", default=os.environ.get("DK_LIB_PATH", "tree"))
    ap.add_argument("--events", action="store_true", help="record events around every launch")
    ap.add_argument("--ring", type=int, default=1, help="distinct action/output buffers")
    a = ap.parse_args()
    import torch

    import paper_2502_08844_b200 as dk

    res = []
    for n in [int(x) for x in a.worlds.split(",")]:
        env = dk.DeviceBatchEnv(dk.EnvConfig(task=a.task), n, dtype=a.dtype)
        env.reset(seed=0)
        acts_r = [torch.rand((a.steps, n, env.action_dim), device="cuda", dtype=env.dtype) * 2 - 1
                  for _ in range(a.ring)]
        out_r = [env._outputs((a.steps,), True) for _ in range(a.ring)]
        acts, out = acts_r[0], out_r[0]
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(2 * a.launches)]
        for _ in range(3):
            env.rollout(acts, with_info=True, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        import time
        e0.record()
        h0 = time.perf_counter()
        for L in range(a.launches):
            if a.events:
                evs[2 * L].record()
            env.rollout(acts_r[L % a.ring], with_info=True, out=out_r[L % a.ring])
            if a.events:
                evs[2 * L + 1].record()
        host_us = (time.perf_counter() - h0) * 1e6 / a.launches
        e1.record()
        torch.cuda.synchronize()
        env.check()
        ms = e0.elapsed_time(e1)
        ns_step = ms * 1e6 / (a.launches * a.steps)
        res.append(f"{n}:{ns_step:.1f}ns/{n / ns_step:.3g}e9(host {host_us:.0f}us/call)")
    print(os.path.basename(a.tag), a.dtype, " ".join(res))


if __name__ == "__main__":
    main()
