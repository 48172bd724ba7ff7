"""Rollout-side PPO math on the GPU.

Mirrors of the reference functions that run on every rollout batch, over CUDA
tensors through the C ABI (include/deskrl_b200.h):

* ``compute_gae_batch`` -- ``ppo.compute_gae`` (ppo.py:80-102): advantages and
  value targets from time-major [T, N] rewards / values / dones and the [N]
  bootstrap values;
* ``DeviceRunningNormalizer`` -- ``mathcore.RunningNormalizer`` with
  ``normalizer_update`` / ``normalizer_apply`` / ``normalizer_invert``
  (mathcore.py:218-272): statistics kept on the device in float64.

All arithmetic is float64 in the reference's operation order whatever the
storage dtype (the reference converts its inputs with ``np.asarray(float)``);
float32 tensors are rounded once on output.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from .envkit import InvalidInputError, _check


def _torch():
    import torch

    return torch


def _dtype_code(t):
    torch = _torch()
    if t.dtype == torch.float64:
        return nat.DK_F64
    if t.dtype == torch.float32:
        return nat.DK_F32
    raise InvalidInputError(f"unsupported dtype {t.dtype} (float32 or float64)")


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(dev):
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def compute_gae_batch(rewards, values, bootstrap, dones, gamma: float, lam: float):
    """ppo.compute_gae on CUDA tensors: returns (advantages, returns) [T, N]."""
    torch = _torch()
    r = rewards.contiguous()
    dt = r.dtype
    v = values.to(dt).contiguous()
    d = dones.to(dt).contiguous()
    if r.shape != v.shape or r.shape != d.shape:
        raise InvalidInputError("compute_gae: mismatched shapes")
    if r.dim() == 1:
        r, v, d = r[:, None], v[:, None], d[:, None]
    T = r.shape[0]
    N = r.numel() // max(T, 1)
    b = torch.as_tensor(bootstrap, device=r.device).to(dt).reshape(-1).contiguous()
    if b.numel() != N:
        raise InvalidInputError("compute_gae: mismatched shapes")
    adv = torch.empty_like(r)
    ret = torch.empty_like(r)
    _check(nat.lib().dk_ppo_gae(_dtype_code(r), T, N, _ptr(r), _ptr(v), _ptr(d), _ptr(b),
                                float(gamma), float(lam), _ptr(adv), _ptr(ret),
                                _stream(r.device)))
    shape = rewards.shape
    return adv.reshape(shape), ret.reshape(shape)


class DeviceRunningNormalizer:
    """mathcore.RunningNormalizer with float64 statistics on the device."""

    def __init__(self, dim: int, epsilon: float = 1e-8, device=None, count: float = 0.0,
                 mean=None, var=None):
        torch = _torch()
        self.dim = int(dim)
        self.epsilon = float(epsilon)
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)
        self.count = float(count)
        self.mean = (torch.zeros(dim, dtype=torch.float64, device=self.device) if mean is None
                     else torch.as_tensor(mean, dtype=torch.float64, device=self.device).clone())
        self.var = (torch.zeros(dim, dtype=torch.float64, device=self.device) if var is None
                    else torch.as_tensor(var, dtype=torch.float64, device=self.device).clone())

    @classmethod
    def from_reference(cls, n, device=None):
        return cls(n.dim, n.epsilon, device, n.count, np.asarray(n.mean), np.asarray(n.var))

    def to_numpy(self):
        """(count, mean, var) as the reference's RunningNormalizer fields."""
        return self.count, self.mean.cpu().numpy(), self.var.cpu().numpy()

    def _rows(self, batch):
        b = batch if batch.dim() > 1 else batch[None]
        if b.shape[-1] != self.dim:
            raise InvalidInputError(
                f"normalizer dim mismatch: expected {self.dim}, got {b.shape[-1]}")
        return b.reshape(-1, self.dim).contiguous()

    def update(self, batch, dist=None, group=None):
        """normalizer_update: merge the rows of ``batch`` (float32/64 CUDA tensor).

        With an initialised ``torch.distributed`` (``dist``) of several ranks,
        the merged batch is the concatenation of every rank's rows, as if one
        process had called normalizer_update on all of them (the
        rollout-statistic reduction): column sums, then squared deviations
        from the global mean, are all-reduced (NCCL between GPUs) and every
        rank applies the same merge.  Tree / rank summation order: 1e-13."""
        torch = _torch()
        b = self._rows(batch)
        rows = b.shape[0]
        st = _stream(b.device)
        lib = nat.lib()
        # scratch from torch's caching allocator (stream-ordered, reused)
        wsb = int(lib.dk_norm_workspace_bytes(rows, self.dim))
        ws = torch.empty(max(wsb, 8), dtype=torch.uint8, device=b.device)
        if dist is None or not dist.is_initialized() or dist.get_world_size(group) == 1:
            _check(lib.dk_norm_update(_dtype_code(b), rows, self.dim, _ptr(b), self.count,
                                      _ptr(self.mean), _ptr(self.var), _ptr(ws), wsb, st))
            self.count += rows
            return self
        n = torch.tensor([float(rows)], dtype=torch.float64, device=b.device)
        dist.all_reduce(n, group=group)
        total = float(n.item())
        sums = torch.empty(self.dim, dtype=torch.float64, device=b.device)
        _check(lib.dk_norm_colsum(_dtype_code(b), rows, self.dim, _ptr(b), None, _ptr(sums),
                                  _ptr(ws), wsb, st))
        dist.all_reduce(sums, group=group)
        b_mean = sums / total
        sq = torch.empty_like(sums)
        _check(lib.dk_norm_colsum(_dtype_code(b), rows, self.dim, _ptr(b), _ptr(b_mean),
                                  _ptr(sq), _ptr(ws), wsb, st))
        dist.all_reduce(sq, group=group)
        b_var = sq / total
        _check(lib.dk_norm_merge(self.dim, self.count, total, _ptr(b_mean), _ptr(b_var),
                                 _ptr(self.mean), _ptr(self.var), st))
        self.count += total
        return self

    def _apply(self, batch, invert):
        if batch.shape[-1] != self.dim:
            raise InvalidInputError(
                f"normalizer dim mismatch: expected {self.dim}, got {batch.shape[-1]}")
        b = batch.contiguous()
        out = _torch().empty_like(b)
        _check(nat.lib().dk_norm_apply(_dtype_code(b), b.numel() // self.dim, self.dim, _ptr(b),
                                       self.count, _ptr(self.mean), _ptr(self.var), self.epsilon,
                                       int(invert), _ptr(out), _stream(b.device)))
        return out

    def apply(self, batch):
        """normalizer_apply: clip((x - mean) / sqrt(var + eps), -10, 10)."""
        return self._apply(batch, False)

    def invert(self, batch):
        """normalizer_invert: x * sqrt(var + eps) + mean."""
        return self._apply(batch, True)


__all__ = ["DeviceRunningNormalizer", "compute_gae_batch"]
