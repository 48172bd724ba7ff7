"""The PPO networks' MLP forward on the B200 tensor cores (csrc/mlp_tc.cuh,
C ABI dk_mlp_*): SURVEY.md §8f rank 1, reference ppo.py:109-141 (_mlp,
MLPPolicy, MLPValue: Linear + Swish layers).

``TensorCoreMLP(seq)`` wraps a torch ``nn.Sequential`` of the reference's shape
-- Linear(d_in, H), SiLU, [Linear(H, H), SiLU] x n, Linear(H, n_out) with
H in {128, 256}, d_in <= 128, n_out <= 16 -- and evaluates it in one kernel:
layer 0 and the output layer in float32 on the CUDA cores, the H x H layers
on tcgen05 with a BF16x3 operand split (float32 accumulation; ~1e-6 relative
to a float32 evaluation).  The packed weights are rebuilt when a parameter
changes (torch's per-tensor version counters).  ``tc_policy`` / ``tc_value``
wrap the reference's MLPPolicy / MLPValue (same outputs: (mean, log_std) and
value).  No CPU path: the kernel needs an sm_100a GPU.
"""

from __future__ import annotations

import ctypes

from . import _native as nat
from .envkit import ConfigError, _check


class MlpC(ctypes.Structure):
    _fields_ = [("d_in", ctypes.c_int32), ("hidden", ctypes.c_int32), ("n_tc", ctypes.c_int32),
                ("n_out", ctypes.c_int32), ("w0", ctypes.c_void_p), ("b0", ctypes.c_void_p),
                ("w_hi", ctypes.c_void_p), ("w_lo", ctypes.c_void_p),
                ("b_hidden", ctypes.c_void_p), ("w_out", ctypes.c_void_p),
                ("b_out", ctypes.c_void_p), ("w0_hi", ctypes.c_void_p),
                ("w0_lo", ctypes.c_void_p)]


def _linears(seq):
    import torch.nn as nn

    mods = list(seq)
    lins = [m for m in mods if isinstance(m, nn.Linear)]
    acts = [m for m in mods if not isinstance(m, nn.Linear)]
    if not all(isinstance(a, nn.SiLU) for a in acts) or len(acts) != len(lins) - 1:
        raise ConfigError("TensorCoreMLP: expected Linear / SiLU alternating, ending in Linear")
    for i, m in enumerate(mods):
        if isinstance(m, nn.Linear) != (i % 2 == 0):
            raise ConfigError("TensorCoreMLP: expected Linear / SiLU alternating")
    return lins


def supported(seq) -> bool:
    import torch.nn as nn

    if not isinstance(seq, nn.Sequential):
        return False
    try:
        lins = _linears(seq)
    except ConfigError:
        return False
    if len(lins) < 3:
        return False
    H = lins[0].out_features
    hidden = lins[1:-1]
    return (H in (128, 256) and lins[0].in_features <= 128 and lins[-1].out_features <= 16
            and all(m.in_features == H and m.out_features == H for m in hidden)
            and lins[-1].in_features == H and all(m.bias is not None for m in lins))


class TensorCoreMLP:
    def __init__(self, seq, desc_swap: int = 0):
        import torch

        self._torch = torch
        if not supported(seq):
            raise ConfigError("TensorCoreMLP: unsupported network shape")
        self.seq = seq
        self.lins = _linears(seq)
        self.d_in = self.lins[0].in_features
        self.H = self.lins[0].out_features
        self.n_tc = len(self.lins) - 2
        self.n_out = self.lins[-1].out_features
        self.desc_swap = int(desc_swap)
        self._lib = nat.lib()
        self._key = None
        self.packs = 0

    def _params_key(self):
        return tuple((p.data_ptr(), p._version) for m in self.lins for p in (m.weight, m.bias))

    def _pack(self):
        torch = self._torch
        key = self._params_key()
        if key == self._key:
            return
        dev = self.lins[0].weight.device
        H, n = self.H, self.n_tc
        f32 = lambda t: t.detach().to(torch.float32).contiguous()  # noqa: E731
        self.w0, self.b0 = f32(self.lins[0].weight), f32(self.lins[0].bias)
        self.w_hi = torch.empty((n, H * H), dtype=torch.bfloat16, device=dev)
        self.w_lo = torch.empty((n, H * H), dtype=torch.bfloat16, device=dev)
        self._hid_w = [f32(m.weight) for m in self.lins[1:-1]]
        stream = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
        for i, w in enumerate(self._hid_w):
            _check(self._lib.dk_mlp_pack(w.data_ptr(), H, H, self.w_hi[i].data_ptr(),
                                         self.w_lo[i].data_ptr(), stream))
        self.b_h = torch.stack([f32(m.bias) for m in self.lins[1:-1]]).contiguous()
        self.w_out, self.b_out = f32(self.lins[-1].weight), f32(self.lins[-1].bias)
        w0p = [None, None]
        if self.d_in > 16:  # layer 0 on the tensor cores: packed, K padded to 32
            k0 = (self.d_in + 31) // 32 * 32
            w0pad = torch.zeros((H, k0), dtype=torch.float32, device=dev)
            w0pad[:, :self.d_in] = self.w0
            self.w0_hi = torch.empty((H * k0,), dtype=torch.bfloat16, device=dev)
            self.w0_lo = torch.empty((H * k0,), dtype=torch.bfloat16, device=dev)
            _check(self._lib.dk_mlp_pack(w0pad.data_ptr(), H, k0, self.w0_hi.data_ptr(),
                                         self.w0_lo.data_ptr(), stream))
            self._w0pad = w0pad
            w0p = [self.w0_hi.data_ptr(), self.w0_lo.data_ptr()]
        self._net = MlpC(self.d_in, H, n, self.n_out, self.w0.data_ptr(), self.b0.data_ptr(),
                         self.w_hi.data_ptr(), self.w_lo.data_ptr(), self.b_h.data_ptr(),
                         self.w_out.data_ptr(), self.b_out.data_ptr(), w0p[0], w0p[1])
        self._key = key
        self.packs += 1

    def __call__(self, x):
        torch = self._torch
        self._pack()
        x2 = x.reshape(-1, x.shape[-1])
        if x2.dtype != torch.float32 or x2.stride(-1) != 1:
            x2 = x2.to(torch.float32).contiguous()
        rows = x2.shape[0]
        y = torch.empty((rows, self.n_out), dtype=torch.float32, device=x2.device)
        stream = ctypes.c_void_p(torch.cuda.current_stream(x2.device).cuda_stream)
        _check(self._lib.dk_mlp_forward_dbg(ctypes.byref(self._net), rows, x2.data_ptr(),
                                            x2.stride(0), y.data_ptr(), y.stride(0),
                                            self.desc_swap, stream))
        return y.reshape(*x.shape[:-1], self.n_out)

    def forward_count(self, x, count):
        """Rows [0, *count) of x [R, d_in] (count: a 1-element int64 CUDA tensor
        written by an earlier kernel on the stream); y [R, n_out], rows past the
        count untouched."""
        torch = self._torch
        self._pack()
        if x.dtype != torch.float32 or x.stride(-1) != 1 or x.dim() != 2:
            raise ConfigError("forward_count: x must be a 2-D float32 row-major tensor")
        rows = x.shape[0]
        y = torch.empty((rows, self.n_out), dtype=torch.float32, device=x.device)
        stream = ctypes.c_void_p(torch.cuda.current_stream(x.device).cuda_stream)
        _check(self._lib.dk_mlp_forward_count(ctypes.byref(self._net), rows, count.data_ptr(),
                                              x.data_ptr(), x.stride(0), y.data_ptr(),
                                              y.stride(0), stream))
        return y


def forward_pair(m0, x0, m1, x1):
    """Two TensorCoreMLP forwards in one launch (dk_mlp_forward_pair): the
    networks' row tiles run side by side.  x0 / x1: 2-D float32 row-major CUDA
    tensors on one device.  Returns (y0, y1)."""
    torch = m0._torch
    m0._pack()
    m1._pack()
    for x in (x0, x1):
        if x.dtype != torch.float32 or x.dim() != 2 or x.stride(-1) != 1:
            raise ConfigError("forward_pair: inputs must be 2-D float32 row-major tensors")
    y0 = torch.empty((x0.shape[0], m0.n_out), dtype=torch.float32, device=x0.device)
    y1 = torch.empty((x1.shape[0], m1.n_out), dtype=torch.float32, device=x1.device)
    stream = ctypes.c_void_p(torch.cuda.current_stream(x0.device).cuda_stream)
    _check(m0._lib.dk_mlp_forward_pair(
        ctypes.byref(m0._net), x0.shape[0], x0.data_ptr(), x0.stride(0), y0.data_ptr(),
        y0.stride(0), ctypes.byref(m1._net), x1.shape[0], x1.data_ptr(), x1.stride(0),
        y1.data_ptr(), y1.stride(0), stream))
    return y0, y1


class _TCPolicy:
    """MLPPolicy.forward on the tensor cores: (mean, log_std.expand_as(mean))."""

    def __init__(self, policy):
        self.module = policy
        self.mlp = TensorCoreMLP(policy.trunk)
        self.action_dim = policy.action_dim

    def __call__(self, obs):
        mean = self.mlp(obs)
        return mean, self.module.log_std.expand_as(mean)

    def parameters(self):
        return self.module.parameters()


class _TCValue:
    """MLPValue.forward on the tensor cores: trunk(obs).squeeze(-1)."""

    def __init__(self, value):
        self.module = value
        self.mlp = TensorCoreMLP(value.trunk)

    def __call__(self, obs):
        return self.mlp(obs).squeeze(-1)

    def call_count(self, obs, count):
        """values of rows [0, *count) of obs (device-side count)"""
        return self.mlp.forward_count(obs, count).squeeze(-1)

    def parameters(self):
        return self.module.parameters()


def tc_policy(policy):
    """Tensor-core forward for a reference-shaped MLPPolicy (or the module
    itself when its shape is not supported)."""
    return _TCPolicy(policy) if hasattr(policy, "trunk") and supported(policy.trunk) else policy


def tc_value(value):
    return _TCValue(value) if hasattr(value, "trunk") and supported(value.trunk) else value


__all__ = ["TensorCoreMLP", "forward_pair", "supported", "tc_policy", "tc_value"]
