"""Time compute_gae_batch and the normaliser update at rollout sizes."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2502_08844_b200 import ppo as P

    n, T = 8192, 1000
    for dt in (torch.float32, torch.float64):
        r = torch.randn((T, n), device="cuda", dtype=dt)
        v = torch.randn((T, n), device="cuda", dtype=dt)
        d = (torch.rand((T, n), device="cuda") < 0.001).to(dt)
        b = torch.randn(n, device="cuda", dtype=dt)
        P.compute_gae_batch(r, v, b, d, 0.99, 0.95)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            P.compute_gae_batch(r, v, b, d, 0.99, 0.95)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        esz = 8 if dt == torch.float64 else 4
        print(f"gae {dt}: {ms:.3f} ms for {T}x{n}: {5 * T * n * esz / ms / 1e6:.0f} GB/s")
        x = torch.randn((30 * n, 75), device="cuda", dtype=dt)
        nz = P.DeviceRunningNormalizer(75)
        nz.update(x)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(5):
            nz.update(x)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(f"norm update {dt}: {ms:.3f} ms for {30 * n}x75: {2 * x.numel() * esz / ms / 1e6:.0f} GB/s (2 passes)")


if __name__ == "__main__":
    main()
