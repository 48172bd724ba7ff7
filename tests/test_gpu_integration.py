"""The integration paths of INTEGRATION.md work as written: the ctypes binding
snippet runs verbatim against libdeskrl_b200.so, and the device API can be
captured in a CUDA graph (launch-bound PPO loops replay it)."""

import os
import re

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_integration_ctypes_snippet_runs(monkeypatch):
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    blocks = re.findall(r"```python\n(.*?)```", text, re.S)
    snippet = [b for b in blocks if "dk_env_create" in b][0]
    monkeypatch.chdir(ROOT)
    ns = {}
    exec(compile(snippet, "INTEGRATION.md", "exec"), ns)
    assert ns["rc"] == 0
    assert np.isfinite(ns["obs"]).all() and ns["obs"].shape == (1024, 5)
    assert (ns["rew"] > 0).all()


def test_device_step_is_cuda_graph_capturable():
    import paper_2502_08844_b200 as dk

    n = 4096
    cfg = dk.EnvConfig(task="cartpole-balance", episode_length=7)
    eager = dk.DeviceBatchEnv(cfg, n, dtype="float32")
    graphed = dk.DeviceBatchEnv(cfg, n, dtype="float32")
    acts = [torch.rand((n, 1), device="cuda") * 2 - 1 for _ in range(12)]
    eager.reset(seed=5)
    graphed.reset(seed=5)
    a_buf = torch.zeros((n, 1), device="cuda")
    out = graphed._outputs((), True)
    # warm up on a side stream (first call sets kernel attributes), then capture
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        a_buf.copy_(acts[0])
        graphed.step(a_buf, out=out)
        ref0 = eager.step(acts[0])
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    assert torch.equal(out["obs"], ref0["obs"])
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        graphed.step(a_buf, out=out)
    for k in range(1, 12):
        a_buf.copy_(acts[k])
        g.replay()
        ref = eager.step(acts[k])
        torch.cuda.synchronize()
        assert torch.equal(out["obs"], ref["obs"]), k
        assert torch.equal(out["reward"], ref["reward"]), k
        assert torch.equal(out["trunc"], ref["trunc"]), k
    graphed.check()
    s1, *_ = graphed.state()
    s2, *_ = eager.state()
    np.testing.assert_array_equal(s1, s2)


def test_no_leak_over_create_close_cycles():
    """no leaks over 10^3 create / close cycles of
    the bindings handle (device memory and pinned host staging)."""
    import torch

    import paper_2502_08844_b200 as dk

    def cycle(k):
        for _ in range(k):
            env = dk.BatchEnv(dk.EnvConfig(task="cartpole-balance"), 64)
            env.reset(seed=1)
            env.step(np.zeros((64, 1)))
            env.close()

    cycle(20)
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()
    cycle(1000)
    torch.cuda.synchronize()
    free1, _ = torch.cuda.mem_get_info()
    assert free0 - free1 < 4 * 1024 * 1024, (free0, free1)
