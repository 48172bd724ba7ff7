"""Time the fused Go1-shape step tail with and without observation noise
(Philox share of the kernel).  python tools/exp_tail.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    from paper_2502_08844_b200 import locomotion as L

    n, K = 8192, 100
    for dt in (torch.float32,):
        fr = bench.synthetic_frames(K * n, 12, 4, torch.device("cuda"), dt, 1)
        for label, noise in (("noise", L.ObservationNoise(0.05, 0.1, 0.2, 0.01, 1.5)),
                             ("no-noise", None)):
            def run(j):
                return L.locomotion_tail(fr, noise=noise, key=L.NoiseKey(0, 0, None, j * K),
                                         num_worlds=n, check=False)
            for j in range(3):
                run(j)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for j in range(10):
                run(j)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 10
            print(f"{label}: {ms:.3f} ms per {K}x{n} rows -> {K * n / ms / 1e6:.3g}e9 rows/s, "
                  f"{K * n * 993 / ms / 1e6:.0f} GB/s")


if __name__ == "__main__":
    main()
