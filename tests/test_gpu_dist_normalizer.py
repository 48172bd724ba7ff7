"""Data-parallel normaliser update (SURVEY §8e rollout-statistic reduction):
two ranks, each with half of the rows, all-reduce column sums and squared
deviations and end with the statistics a single process gets from all rows
(the reference's normalizer_update on the concatenation), to 1e-13.
Both ranks run on GPU 0 over gloo (the round's GPU boxes have one GPU; NCCL
between GPUs is the same call)."""
import os
import tempfile

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _worker(rank, world, init, out_path):
    import torch.distributed as dist

    from paper_2502_08844_b200 import ppo as P

    dist.init_process_group("gloo", init_method=init, rank=rank, world_size=world)
    torch.cuda.set_device(0)
    rng = np.random.default_rng(5)
    x = rng.normal(rng.uniform(-2, 2, 11), rng.uniform(0.1, 3, 11), (3000, 11))
    y = rng.normal(0.5, 1.0, (777, 11))
    n = P.DeviceRunningNormalizer(11)
    for batch in (x, y):
        half = batch[rank::world]
        n.update(torch.as_tensor(half, device="cuda"), dist=dist)
    c, m, v = n.to_numpy()
    np.savez(f"{out_path}.{rank}.npz", count=c, mean=m, var=v)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_update_equals_single_process():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    from oracle import ppo as orc

    with tempfile.TemporaryDirectory() as d:
        init = "file://" + os.path.join(d, "rendezvous")
        out = os.path.join(d, "stats")
        mp.spawn(_worker, args=(2, init, out), nprocs=2, join=True)
        rng = np.random.default_rng(5)
        x = rng.normal(rng.uniform(-2, 2, 11), rng.uniform(0.1, 3, 11), (3000, 11))
        y = rng.normal(0.5, 1.0, (777, 11))
        c, m, v = orc.norm_update(0.0, np.zeros(11), np.zeros(11), x)
        c, m, v = orc.norm_update(c, m, v, y)
        for r in range(2):
            got = np.load(f"{out}.{r}.npz")
            assert float(got["count"]) == c
            np.testing.assert_allclose(got["mean"], m, rtol=1e-13, atol=1e-15)
            np.testing.assert_allclose(got["var"], v, rtol=1e-13)
