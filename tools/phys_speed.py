"""Time the articulated physics kernel: physics steps/s at several world counts
(ctrl held, no diagnostics), f32 and f64.  Not a bench line.

    python tools/phys_speed.py [--worlds 1024,8192,65536] [--steps 100]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--worlds", default="1024,8192,65536")
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--dtypes", default="float32,float64")
    ap.add_argument("--full", action="store_true", help="box + thigh collisions")
    a = ap.parse_args()
    import torch

    from oracle import physics as op
    from paper_2502_08844_b200 import physics as P
    from paper_2502_08844_b200 import physmodel as pm

    model = pm.go1_model(**(dict(collide_box=1, collide_thigh=1) if a.full else {}))
    for dt in a.dtypes.split(","):
        res = []
        for n in [int(x) for x in a.worlds.split(",")]:
            sim = P.DevicePhysics(model, n, dtype=dt)
            qpos, qvel, ctrl = op.random_states(n, seed=1)
            t = lambda x: torch.as_tensor(x, device="cuda", dtype=sim.dtype)  # noqa: E731
            sim.set_state(t(qpos), t(qvel))
            c = t(ctrl)
            sim.step(c, a.steps, diag=False)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            reps = 3
            for _ in range(reps):
                sim.step(c, a.steps, diag=False)
            e1.record()
            torch.cuda.synchronize()
            sim.check()
            ms = e0.elapsed_time(e1) / reps
            res.append(f"{n}:{n * a.steps / (ms / 1e3):.3g}/s({ms:.2f}ms/{a.steps})")
            sim.close()
        print("phys", "full" if a.full else "feet", dt, " ".join(res), flush=True)


if __name__ == "__main__":
    main()
