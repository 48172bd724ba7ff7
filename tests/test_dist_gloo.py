"""Multi-process (world_size 2, gloo, CPU) checks of the sharding logic used by
the multi-GPU path: each rank steps only its block of worlds -- here with the
CPU oracle standing in for the kernel -- keyed by its global env-index offset,
and the gathered result is bit-identical to one unsharded run (the
worker-count invariance of SPEC.md:282/785, extended to ranks)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, K, out_path):
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import OracleBatchEnv
    from paper_2502_08844_b200.distributed import max_over_ranks, shard, sum_over_ranks

    off, cnt = shard(n, rank, world)
    acts = np.random.default_rng(3).uniform(-1, 1, (K, n, 1))
    env = OracleBatchEnv("cartpole-balance", cnt, episode_length=40, env_offset=off)
    env.reset(seed=9)
    obs, rew, done, trunc, *_ = env.rollout(acts[:, off:off + cnt])
    parts = [None] * world
    dist.all_gather_object(parts, (off, obs, rew, trunc, env.state))
    t = max_over_ranks(1.0 + rank, dist)
    s = sum_over_ranks(cnt, dist)
    if rank == 0:
        parts.sort(key=lambda p: p[0])
        np.savez(out_path, obs=np.concatenate([p[1] for p in parts], 1),
                 rew=np.concatenate([p[2] for p in parts], 1),
                 trunc=np.concatenate([p[3] for p in parts], 1),
                 state=np.concatenate([p[4] for p in parts], 0), tmax=t, total=s)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [64, 67])
def test_two_rank_shards_equal_single_run(tmp_path, oracle, n):
    K = 90
    out = tmp_path / "gathered.npz"
    mp.spawn(_worker, args=(2, _free_port(), n, K, str(out)), nprocs=2, join=True)
    g = np.load(out)
    ref = oracle.OracleBatchEnv("cartpole-balance", n, episode_length=40)
    ref.reset(seed=9)
    acts = np.random.default_rng(3).uniform(-1, 1, (K, n, 1))
    obs, rew, done, trunc, *_ = ref.rollout(acts)
    np.testing.assert_array_equal(g["obs"], obs)
    np.testing.assert_array_equal(g["rew"], rew)
    np.testing.assert_array_equal(g["trunc"], trunc)
    np.testing.assert_array_equal(g["state"], ref.state)
    assert float(g["tmax"]) == 2.0 and int(g["total"]) == n


def test_shard_partition():
    from paper_2502_08844_b200.distributed import shard

    for n in (1, 7, 8192, 10001):
        for w in (1, 2, 3, 8):
            blocks = [shard(n, r, w) for r in range(w)]
            assert blocks[0][0] == 0
            assert sum(c for _, c in blocks) == n
            for (o1, c1), (o2, _) in zip(blocks, blocks[1:]):
                assert o1 + c1 == o2
