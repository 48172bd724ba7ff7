"""World sharding across ranks through the real kernels: two
gloo ranks, both on GPU 0 (the kernels of the two ranks never wait on each
other), each stepping its shard [r*N, (r+1)*N) of the worlds with
env_index_offset; the gathered trajectories equal one process stepping all
2N worlds bit for bit (Philox streams are keyed by the global world index).
Covers the analytic env (DeviceBatchEnv) and the fused Go1 joystick env."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, K, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2502_08844_b200 as dk
        from paper_2502_08844_b200 import go1env as G

        torch.cuda.set_device(0)
        acts = torch.as_tensor(np.random.default_rng(3).uniform(-1, 1, (K, world * n, 1)))
        env = dk.DeviceBatchEnv(dk.EnvConfig(task="cartpole-balance", episode_length=7), n,
                                dtype="float64", env_index_offset=rank * n)
        env.reset(seed=9)
        o = env.rollout(acts[:, rank * n:(rank + 1) * n].cuda())
        env.check()
        parts = [torch.zeros((K, n, 5), dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, o["obs"].cpu())
        ga = torch.as_tensor(np.random.default_rng(4).uniform(-1, 1, (K, world * n, 12)))
        genv = G.DeviceGo1Env(n, G.Go1Config(episode_length=5, seed=2), dtype="float64",
                              env_index_offset=rank * n)
        genv.reset()
        go = genv.rollout(ga[:, rank * n:(rank + 1) * n].cuda())
        genv.check()
        gparts = [torch.zeros((K, n, 56), dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gparts, go["obs"].cpu())
        if rank == 0:
            q.put((torch.cat(parts, 1).numpy(), torch.cat(gparts, 1).numpy()))
    finally:
        dist.destroy_process_group()


def test_two_gloo_ranks_equal_one_process():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    import paper_2502_08844_b200 as dk
    from paper_2502_08844_b200 import go1env as G

    n, K, world = 96, 12, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, K, q)) for r in range(world)]
    for p in procs:
        p.start()
    sharded, gsharded = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    acts = torch.as_tensor(np.random.default_rng(3).uniform(-1, 1, (K, world * n, 1))).cuda()
    env = dk.DeviceBatchEnv(dk.EnvConfig(task="cartpole-balance", episode_length=7), world * n,
                            dtype="float64")
    env.reset(seed=9)
    full = env.rollout(acts)["obs"].cpu().numpy()
    np.testing.assert_array_equal(sharded, full)
    ga = torch.as_tensor(np.random.default_rng(4).uniform(-1, 1, (K, world * n, 12))).cuda()
    genv = G.DeviceGo1Env(world * n, G.Go1Config(episode_length=5, seed=2), dtype="float64")
    genv.reset()
    gfull = genv.rollout(ga)["obs"].cpu().numpy()
    np.testing.assert_array_equal(gsharded, gfull)
