"""Break down one pixel-policy rollout step at 8192 worlds (CUDA events):
env step (+render), pixel_normalize, CNN policy forward, value MLP."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2502_08844_b200 as dk  # noqa: E402
from paper_2502_08844_b200 import rollout as R  # noqa: E402
from paper_2502_08844_b200.pixels import pixel_normalize  # noqa: E402

n = 8192
env = dk.DeviceBatchEnv(dk.EnvConfig(task="cartpole-balance-pixels", visual_randomization=True), n)
obs = env.reset(seed=0)
policy = R.make_cnn_policy(3, 64, 1).cuda()
value = R.make_value(5).cuda()
a = torch.zeros(n, 1, device="cuda")
out = env._outputs((), False)


def timeit(name, fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name:40s} {e0.elapsed_time(e1) / reps:8.3f} ms")


x = pixel_normalize(obs["pixels"])
with torch.no_grad():
    timeit("env.step (+render, stack)", lambda: env.step(a, with_info=False, out=out))
    timeit("pixel_normalize", lambda: pixel_normalize(out["pixels"]))
    timeit("CNN policy fwd (tf32 default)", lambda: policy(x))
    torch.backends.cudnn.allow_tf32 = False
    timeit("CNN policy fwd (fp32, tf32 off)", lambda: policy(x))
    torch.backends.cudnn.allow_tf32 = True
    xc = x.contiguous(memory_format=torch.channels_last)
    pc = R.make_cnn_policy(3, 64, 1).cuda().to(memory_format=torch.channels_last)
    timeit("CNN policy fwd (channels_last)", lambda: pc(xc))
    xn = pixel_normalize(obs["pixels"], channels_first=False).permute(0, 3, 1, 2)
    timeit("CNN fwd (NHWC normalize, NCHW weights)", lambda: policy(xn))
    timeit("normalize NHWC + CNN fwd", lambda: policy(
        pixel_normalize(out["pixels"], channels_first=False).permute(0, 3, 1, 2)))
    print("max |NCHW - channels_last| policy mean:",
          float((policy(x)[0] - policy(xn)[0]).abs().max()))
    torch.backends.cudnn.benchmark = True
    timeit("CNN policy fwd (cudnn.benchmark)", lambda: policy(x))
    s = obs["state"].float()
    timeit("value MLP fwd", lambda: value(s))
    timeit("stack clone", lambda: out["pixels"].clone())
