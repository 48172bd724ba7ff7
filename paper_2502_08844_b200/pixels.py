"""Cartpole pixel observations on the GPU.

Mirrors ``pixelrender`` (pixelrender.py:20-186) and the pixel branch of
``Environment.reset`` / ``_observe`` (envkit.py:515-518, 555-577):

* ``batch_render`` -- the orthographic rasteriser (+ ``brightness_postprocess``),
  RGB uint8 [n, h, w, 3];
* ``PixelObservation`` -- the per-world 3-frame grayscale stack that
  ``cartpole-balance-pixels`` returns as ``obs["pixels"]``, including visual
  domain randomisation at reset (``randomize_visuals`` drawn from the episode's
  ``stream_rng`` after ``sample_initial``'s four draws) and the terminal stack of
  autoreset worlds.

A frame is a function of (cart x, cos th, sin th) and the world's visuals, so
the stack is re-rendered from the last three states (write-only HBM traffic)
instead of being read back.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from .envkit import ConfigError, InvalidInputError, _check

# VisualParams() / VisualBounds() defaults (pixelrender.py:23-51)
NOMINAL = (40.0, 40.0, 60.0, 200.0, 60.0, 60.0, 240.0, 240.0, 100.0, 0.0, 0.0, 1.0, 1.0)
SAMPLE_INITIAL_WORDS = 4  # cartpole sample_initial: four uniform draws (envkit.py:302-309)


def _torch():
    import torch

    return torch


def pack_visuals(v) -> tuple:
    """VisualParams -> the 13 packed doubles."""
    return (*map(float, v.background), *map(float, v.cart_color), *map(float, v.pole_color),
            float(v.camera_offset[0]), float(v.camera_offset[1]), float(v.camera_zoom),
            float(v.brightness))


def _bounds(nominal=NOMINAL, color_jitter=40.0, camera_offset_range=0.2, zoom_range=(0.85, 1.15),
            brightness_range=(0.7, 1.3)):
    b = nat.VisualBoundsC()
    for k, x in enumerate(nominal):
        b.nominal[k] = float(x)
    b.color_jitter, b.camera_offset_range = float(color_jitter), float(camera_offset_range)
    b.zoom_range[0], b.zoom_range[1] = map(float, zoom_range)
    b.brightness_range[0], b.brightness_range[1] = map(float, brightness_range)
    return b


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(dev):
    return ctypes.c_void_p(_torch().cuda.current_stream(dev).cuda_stream)


def _dtype_code(t):
    torch = _torch()
    return nat.DK_F64 if t.dtype == torch.float64 else nat.DK_F32


def batch_render(frames, visuals, w: int, h: int, pole_length: float = 0.5,
                 brightness: bool = False):
    """pixelrender.batch_render: frames [n, 3] (x, cos th, sin th) and visuals
    [n, 13] CUDA float64 -> RGB [n, h, w, 3] uint8 (brightness_postprocess
    applied when ``brightness``)."""
    torch = _torch()
    if w <= 0 or h <= 0:
        raise InvalidInputError("viewport must have positive area")
    f = frames.to(torch.float64).contiguous()
    v = visuals.to(torch.float64).contiguous()
    if v.shape != (f.shape[0], 13):
        raise InvalidInputError("params length must match batch size")
    out = torch.empty((f.shape[0], h, w, 3), dtype=torch.uint8, device=f.device)
    _check(nat.lib().dk_pixels_render_rgb(f.shape[0], w, h, float(pole_length), _ptr(f), _ptr(v),
                                          int(bool(brightness)), _ptr(out), _stream(f.device)))
    return out


class PixelObservation:
    """The ``obs["pixels"]`` stacks of ``num_envs`` cartpole worlds on the GPU."""

    def __init__(self, num_envs: int, image_size: int = 64, visual_randomization: bool = False,
                 seed: int = 0, env_index_offset: int = 0, pole_length: float = 0.5,
                 dtype=None, device=None):
        torch = _torch()
        if image_size <= 0:
            raise InvalidInputError("viewport must have positive area")
        self.n, self.size = int(num_envs), int(image_size)
        self.randomize = bool(visual_randomization)
        self.seed, self.env0 = int(seed), int(env_index_offset)
        self.pole_length = float(pole_length)
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)
        self.dtype = dtype or torch.float32
        self.history = torch.zeros((self.n, 3, 3), dtype=torch.float64, device=self.device)
        self.visuals = torch.zeros((self.n, 13), dtype=torch.float64, device=self.device)
        self.episode = torch.zeros(self.n, dtype=torch.int32, device=self.device)
        self._bounds = _bounds()
        self._ready = False

    def _stack(self):
        torch = _torch()
        out = torch.empty((self.n, self.size, self.size, 3), dtype=self.dtype, device=self.device)
        _check(nat.lib().dk_pixels_stack(_dtype_code(out), self.n, self.size, self.size,
                                         self.pole_length, _ptr(self.history),
                                         _ptr(self.visuals), _ptr(out), _stream(self.device)))
        return out

    def _advance(self, obs, mask, first):
        o = obs.contiguous()
        _check(nat.lib().dk_pixels_advance(
            _dtype_code(o), self.n, o.shape[-1], _ptr(o), _ptr(mask), int(first),
            _ptr(self.history), _ptr(self.visuals), _ptr(self.episode), int(self.randomize),
            ctypes.byref(self._bounds), self.seed & (2**64 - 1), self.env0,
            SAMPLE_INITIAL_WORDS, _stream(self.device)))

    def reset(self, obs, seed: int | None = None):
        """After BatchEnv.reset: ``obs`` = the state observations [n, 5].  A new
        ``seed`` rewinds every world to episode 0 (envkit.py:503-505), otherwise
        each world starts its next episode."""
        if seed is not None:
            self.seed = int(seed)
            self.episode.zero_()
        elif self._ready:
            self.episode += 1
        self._advance(obs.to(self.dtype), None, True)
        self._ready = True
        return self._stack()

    def step(self, step_out: dict, terminal: bool = True):
        """After DeviceBatchEnv.step (autoreset): returns (pixels [n, s, s, 3],
        terminal pixels or None).  Rows of the terminal tensor are meaningful
        where ``step_out["terminal_mask"]``."""
        if not self._ready:
            raise InvalidInputError("frame stack read before reset")
        torch = _torch()
        mask = step_out["terminal_mask"].to(torch.uint8).contiguous()
        term = None
        if terminal:
            term = torch.empty((self.n, self.size, self.size, 3), dtype=self.dtype,
                               device=self.device)  # rows written where the mask is set
            t_obs = step_out["terminal_obs"].to(self.dtype).contiguous()
            _check(nat.lib().dk_pixels_terminal(
                _dtype_code(term), self.n, self.size, self.size, self.pole_length,
                t_obs.shape[-1], _ptr(t_obs), _ptr(mask), _ptr(self.history), _ptr(self.visuals),
                _ptr(term), _stream(self.device)))
        self._advance(step_out["obs"].to(self.dtype), mask, False)
        return self._stack(), term


def pixel_normalize(x, channels_first: bool = True, out_dtype=None):
    """ppo.pixel_normalize (ppo.py:232-238) on a CUDA [n, h, w, c] stack:
    per-sample, per-channel (x - mean) / std over the pixels (0 where std is
    0), computed in float64 in NumPy's summation order.  Default output: the
    policy's input, float32 [n, c, h, w] (ppo.py:281-283); channels_first=False
    and out_dtype=torch.float64 give NumPy's own result."""
    torch = _torch()
    if x.dim() != 4:
        raise InvalidInputError("pixel_normalize expects [n, h, w, c]")
    if x.dtype not in (torch.float32, torch.float64):
        # the reference accepts any array (uint8 frames, halves): NumPy's mean /
        # std promote to float64; float32 holds every uint8 / half value exactly
        x = x.to(torch.float64 if x.dtype in (torch.int32, torch.int64) else torch.float32)
    x = x.contiguous()
    n, h, w, c = x.shape
    od = out_dtype or torch.float32
    out = torch.empty((n, c, h, w) if channels_first else (n, h, w, c), dtype=od,
                      device=x.device)
    stats = torch.empty((n, c, 2), dtype=torch.float64, device=x.device)
    _check(nat.lib().dk_pixels_normalize(_dtype_code(x), nat.DK_F64 if od == torch.float64
                                         else nat.DK_F32, n, h, w, c, _ptr(x),
                                         int(bool(channels_first)), _ptr(stats), _ptr(out),
                                         _stream(x.device)))
    return out


__all__ = ["NOMINAL", "PixelObservation", "batch_render", "pack_visuals", "pixel_normalize"]
