"""Golden vectors for the rollout-side PPO math, produced by the reference itself.

    python tests/golden/make_golden_ppo.py      (needs /root/reference; CPU)

Calls deskrl.ppo.compute_gae (ppo.py:80-102) and deskrl.mathcore's
RunningNormalizer / normalizer_update / normalizer_apply / normalizer_invert
(mathcore.py:218-272) on seeded random inputs with terminal flags, and writes
tests/golden/ppo_golden.npz.
"""
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF)
    from deskrl import mathcore, ppo

    rng = np.random.default_rng(2502)
    data = {}
    for name, (T, N) in {"small": (16, 5), "mid": (200, 333)}.items():
        r = rng.normal(0, 1, (T, N))
        v = rng.normal(0, 2, (T, N))
        d = (rng.uniform(size=(T, N)) < 0.05).astype(np.float64)
        b = rng.normal(0, 1, N)
        adv, ret = ppo.compute_gae(r, v, b, d, 0.97, 0.95)
        for k, a in (("r", r), ("v", v), ("d", d), ("b", b), ("adv", adv), ("ret", ret)):
            data[f"gae/{name}/{k}"] = a
    # normalizer: three updates of growing batches, apply / invert after each
    D = 9
    n = mathcore.RunningNormalizer(D)
    probe = rng.normal(0, 3, (50, D))
    data["norm/probe"] = probe
    data["norm/apply0"] = mathcore.normalizer_apply(n, probe)
    for k, rows in enumerate((7, 1000, 4096)):
        batch = rng.normal(rng.uniform(-2, 2, D), rng.uniform(0.1, 5, D), (rows, D))
        batch[:, 3] = 1.5  # a constant column (zero variance)
        n = mathcore.normalizer_update(n, batch)
        data[f"norm/batch{k}"] = batch
        data[f"norm/count{k}"] = np.array(n.count)
        data[f"norm/mean{k}"] = n.mean
        data[f"norm/var{k}"] = n.var
        data[f"norm/apply{k + 1}"] = mathcore.normalizer_apply(n, probe)
        data[f"norm/invert{k + 1}"] = mathcore.normalizer_invert(n, probe)
    path = os.path.join(OUT, "ppo_golden.npz")
    np.savez_compressed(path, **data)
    print(f"wrote {path} ({os.path.getsize(path)} bytes, {len(data)} arrays)")


if __name__ == "__main__":
    main()
