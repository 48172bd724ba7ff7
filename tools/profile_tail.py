"""ncu driver: a few launches of the fused Go1-shape step tail (bench shape)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    from paper_2502_08844_b200 import locomotion as L

    dt = torch.float64 if "--f64" in sys.argv else torch.float32
    n, K = 8192, 100
    fr = bench.synthetic_frames(K * n, 12, 4, torch.device("cuda"), dt, 1)
    for j in range(3):
        L.locomotion_tail(fr, noise=L.ObservationNoise(0.05, 0.1, 0.2, 0.01, 1.5),
                          key=L.NoiseKey(0, 0, None, j * K), num_worlds=n)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
