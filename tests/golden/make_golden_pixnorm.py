"""Golden vectors for ppo.pixel_normalize (ppo.py:232-238), produced by the reference.

    python tests/golden/make_golden_pixnorm.py     (needs /root/reference; CPU)

Inputs: reference cartpole pixel stacks (pixels_golden.npz), images with
constant channels (std == 0 -> 0), and random float32 / float64 images of
ragged shapes.  Outputs: the float64 [n, h, w, c] result and the policy input
the reference builds from it (_prep_policy_obs, ppo.py:278-283: float32
[n, c, h, w]).
"""
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF)
    from deskrl import ppo

    px = np.load(os.path.join(OUT, "pixels_golden.npz"))
    rng = np.random.default_rng(232)
    const = rng.uniform(0, 1, (3, 16, 16, 3))
    const[0] = 0.25                 # whole sample constant
    const[1, :, :, 1] = 0.7         # one constant channel
    cases = {
        "stack": px["rand/pixels"][1:4].reshape(-1, 64, 64, 3),
        "const": const,
        "f32": rng.normal(3.0, 2.0, (5, 7, 9, 2)).astype(np.float32),
        "f64": rng.uniform(-1e3, 1e3, (4, 11, 13, 5)),
        "single": rng.uniform(0, 1, (2, 1, 1, 3)),
    }
    data = {}
    for k, x in cases.items():
        y = ppo.pixel_normalize(x)
        data[f"{k}/x"] = x
        data[f"{k}/y"] = y
        data[f"{k}/policy"] = np.ascontiguousarray(np.moveaxis(y, -1, 1)).astype(np.float32)
    path = os.path.join(OUT, "pixnorm_golden.npz")
    np.savez_compressed(path, **data)
    print(f"wrote {path} ({os.path.getsize(path)} bytes, {len(data)} arrays)")


if __name__ == "__main__":
    main()
