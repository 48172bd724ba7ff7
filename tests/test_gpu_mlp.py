"""The PPO networks on the tensor cores (csrc/mlp_tc.cuh, tcgen05 BF16x3):
against a float64 evaluation of the same torch modules (the reference's
ppo.MLPPolicy / MLPValue shapes, ppo.py:109-141).

Tolerance: BF16x3 keeps ~16 significant bits per product with float32
accumulation; outputs agree with float64 to 2e-5 relative to max(|y|, 1) --
the reference itself evaluates these networks in float32 (~1e-6)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def M():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2502_08844_b200 import mlp

    return mlp


def _err(y, ref):
    y, ref = y.detach().double().cpu().numpy(), ref.detach().double().cpu().numpy()
    return float((np.abs(y - ref) / np.maximum(np.abs(ref), 1.0)).max())


@pytest.mark.parametrize("kind,rows", [("policy", 8192), ("value", 8192), ("policy", 1000),
                                       ("value", 77)])
def test_tc_mlp_matches_float64(M, kind, rows):
    from paper_2502_08844_b200 import rollout as R

    torch.manual_seed(0)
    net = (R.make_policy(5, 1) if kind == "policy" else R.make_value(5)).cuda()
    x = torch.randn(rows, 5, device="cuda") * 2
    tc = M.tc_policy(net) if kind == "policy" else M.tc_value(net)
    got = tc(x)[0] if kind == "policy" else tc(x)
    ref64 = net.double()(x.double())
    ref = ref64[0] if kind == "policy" else ref64
    net.float()
    err = _err(got, ref)
    print(kind, rows, "max rel err vs float64 %.2e" % err)
    assert err < 2e-5, err
    # the packed weights follow parameter updates
    with torch.no_grad():
        for p in net.parameters():
            p.mul_(0.5)
    got2 = tc(x)[0] if kind == "policy" else tc(x)
    ref2 = net.double()(x.double())
    ref2 = ref2[0] if kind == "policy" else ref2
    net.float()
    assert _err(got2, ref2) < 2e-5
    assert tc.mlp.packs == 2


def test_tc_mlp_layout_check(M):
    """The operand descriptors' leading / stride byte offsets: the product layout
    reproduces the network, the swapped one does not (guards the K-major
    canonical layout against a silent transposition)."""
    from paper_2502_08844_b200 import rollout as R

    torch.manual_seed(1)
    net = R.make_value(5).cuda()
    x = torch.randn(256, 5, device="cuda")
    ref = net.double()(x.double()).squeeze(-1)
    net.float()
    good = M.TensorCoreMLP(net.trunk)(x).squeeze(-1)
    bad = M.TensorCoreMLP(net.trunk, desc_swap=1)(x).squeeze(-1)
    assert _err(good, ref) < 2e-5
    assert _err(bad, ref) > 1e-3


def test_tc_mlp_pair_launch_equals_separate_calls(M):
    """dk_mlp_forward_pair (the PPO policy and value in one launch) gives
    bit-identical outputs to the two separate forwards; the count-limited
    forward (device-side row count) matches on its rows."""
    from paper_2502_08844_b200 import rollout as R

    torch.manual_seed(3)
    pol, val = R.make_policy(5, 1).cuda(), R.make_value(5).cuda()
    tp, tv = M.tc_policy(pol), M.tc_value(val)
    xp, xv = torch.randn(1000, 5, device="cuda"), torch.randn(777, 5, device="cuda")
    yp, yv = M.forward_pair(tp.mlp, xp, tv.mlp, xv)
    torch.testing.assert_close(yp, tp.mlp(xp), rtol=0, atol=0)
    torch.testing.assert_close(yv, tv.mlp(xv), rtol=0, atol=0)
    count = torch.tensor([300], dtype=torch.int64, device="cuda")
    yc = tv.call_count(xv, count)
    torch.testing.assert_close(yc[:300], tv(xv)[:300], rtol=0, atol=0)


@pytest.mark.parametrize("d_in,hidden,n_layers,n_out,rows", [
    (56, 128, 4, 12, 8192),   # a Go1 joystick policy: noisy observation -> 12 joint means
    (75, 256, 5, 1, 3000),    # its critic on the privileged observation
    (17, 128, 3, 16, 129),
    # H = 256 with 16 outputs: a two-stage weight ring (the deepest that fits), with
    # a CUDA-core layer 0 (its weights in the ring's last stage) and a tensor-core one
    (3, 256, 3, 16, 1000),
    (100, 256, 4, 16, 257),
])
def test_tc_mlp_wide_inputs_and_outputs(M, d_in, hidden, n_layers, n_out, rows):
    """d_in > 16 runs layer 0 on the tensor cores too (K padded to 32); up to 16
    outputs; 2-, 3- and 4-stage weight rings (csrc/mlp_tc.cuh mlp_stages): against
    a float64 evaluation."""
    import torch.nn as nn

    torch.manual_seed(d_in)
    mods = [nn.Linear(d_in, hidden), nn.SiLU()]
    for _ in range(n_layers - 2):
        mods += [nn.Linear(hidden, hidden), nn.SiLU()]
    mods += [nn.Linear(hidden, n_out)]
    net = nn.Sequential(*mods).cuda()
    assert M.supported(net)
    tc = M.TensorCoreMLP(net)
    x = torch.randn(rows, d_in, device="cuda") * 2
    got = tc(x)
    ref = net.double()(x.double())
    net.float()
    err = _err(got, ref)
    print(d_in, hidden, n_out, "max rel err vs float64 %.2e" % err)
    assert err < 2e-5, err
