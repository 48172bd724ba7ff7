"""Parity report: B200 env step vs the C oracle (bit-exact restatement of the
reference) for every task and both dtypes, as error-vs-horizon tables.

    python tools/parity_report.py [--out gpurun_out/parity.json]

Error metric per quantity: max |gpu - ref| / max(|ref|, floor) over all
worlds, reported for several floors, at horizons 1, 10, 100, 300, 1000.
Counters and flags are compared exactly.
"""

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

TASKS = ["pendulum-swingup", "cartpole-balance", "acrobot-swingup", "reacher-easy"]
HORIZONS = [1, 10, 100, 300, 1000]
FLOORS = [1e-3, 1e-1, 1.0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "parity.json"))
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--dtypes", default="float64,float32")
    ap.add_argument("--tag", default=os.environ.get("DK_LIB_PATH", "product"))
    args = ap.parse_args()
    import torch

    import paper_2502_08844_b200 as dk
    from oracle.oracle import OracleBatchEnv

    n, K = args.n, max(HORIZONS)
    report = {}
    for task in TASKS:
        A = 2 if task == "reacher-easy" else 1
        acts = np.random.default_rng(42).uniform(-1, 1, (K, n, A))
        for wide in ([False, True] if task == "pendulum-swingup" else [False]):
            ref = OracleBatchEnv(task, n, episode_length=1000, wide_init=wide)
            ref.reset(seed=5)
            r_obs, r_rew, _, r_tr, _, r_mask, r_info = ref.rollout(acts)
            for dtype in args.dtypes.split(","):
                env = dk.DeviceBatchEnv(dk.EnvConfig(task=task, wide_init=wide), n, dtype=dtype)
                env.reset(seed=5)
                out = env.rollout(torch.as_tensor(acts, device="cuda", dtype=env.dtype),
                                  with_info=True)
                env.check()
                obs = out["obs"].double().cpu().numpy()
                rew = out["reward"].double().cpu().numpy()
                tr = out["trunc"].cpu().numpy()
                key = f"{task}{'/wide' if wide else ''}/{dtype}"
                rec = {"trunc_exact": bool(np.array_equal(tr, r_tr)),
                       "mask_exact": bool(np.array_equal(out["terminal_mask"].cpu().numpy(),
                                                         r_mask))}
                for h in HORIZONS:
                    for fl in FLOORS:
                        eo = np.abs(obs[:h] - r_obs[:h]) / np.maximum(np.abs(r_obs[:h]), fl)
                        er = np.abs(rew[:h] - r_rew[:h]) / np.maximum(np.abs(r_rew[:h]), fl)
                        rec[f"obs@{h}/floor{fl:g}"] = float(eo.max())
                        rec[f"rew@{h}/floor{fl:g}"] = float(er.max())
                    rec[f"obs_bitexact_frac@{h}"] = float((obs[:h] == r_obs[:h]).mean())
                    # per observation component, absolute error and rel @ floor 1e-3
                    d = np.abs(obs[:h] - r_obs[:h])
                    rec[f"obs_abs_per_comp@{h}"] = [float(x) for x in d.max(axis=(0, 1))]
                    rec[f"obs_rel_per_comp@{h}/floor0.001"] = [
                        float(x) for x in (d / np.maximum(np.abs(r_obs[:h]), 1e-3)).max(axis=(0, 1))]
                rec["reward_mean_gpu"] = float(rew.mean())
                rec["reward_mean_ref"] = float(r_rew.mean())
                report[key] = rec
                env.close()
                print(key, {k: f"{v:.2e}" if isinstance(v, float) else v for k, v in rec.items()
                            if "floor0.001" in k or "exact" in k}, flush=True)
    report["_tag"] = os.path.basename(args.tag)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(report, f, indent=1)


if __name__ == "__main__":
    main()
