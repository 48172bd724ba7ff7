"""Time pixel_normalize on an [n, 64, 64, 3] float32 stack (CUDA events)."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_08844_b200 import pixels

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
if len(sys.argv) > 2 and sys.argv[2] == "env":  # rendered stacks from the pixel env
    import paper_2502_08844_b200 as dk

    env = dk.DeviceBatchEnv(dk.EnvConfig(task="cartpole-balance-pixels", visual_randomization=True), n)
    env.reset(seed=0)
    for _ in range(3):
        o = env.step(torch.rand(n, 1, device="cuda") * 2 - 1)
    x = o["pixels"].clone()
else:
    x = torch.rand(n, 64, 64, 3, device="cuda")
for _ in range(3):
    pixels.pixel_normalize(x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
R = 20
e0.record()
for _ in range(R):
    pixels.pixel_normalize(x)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / R
alg = 2 * x.numel() * 4  # read once + write once
print(f"n={n} {ms:.3f} ms/call  {alg / ms / 1e6:.0f} GB/s algorithmic")
