"""Time the cartpole pixel env step and its stack kernel alone (8192 worlds, f32)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2502_08844_b200 as dk  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
env = dk.DeviceBatchEnv(dk.EnvConfig(task="cartpole-balance-pixels", visual_randomization=True), n)
env.reset(seed=0)
a = torch.rand(n, 1, device="cuda") * 2 - 1
out = env._outputs((), False)
for _ in range(5):
    env.step(a, with_info=False, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    env._pix._stack()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"stack kernel {ms:.3f} ms  {n * 49152 / ms / 1e6:.0f} GB/s")
