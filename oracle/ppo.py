"""ctypes wrappers of oracle/ppo.c (TEST INFRASTRUCTURE ONLY: tests, smoke, bench).

compute_gae (ppo.py:80-102), pixel_normalize (ppo.py:232-238) and the
RunningNormalizer update / apply / invert
(mathcore.py:234-272) restated in float64."""
import ctypes

import numpy as np

from .oracle import lib as _lib


def _vp(a):
    return ctypes.c_void_p(a.ctypes.data)


def gae(rewards, values, bootstrap, dones, gamma, lam):
    r = np.ascontiguousarray(rewards, dtype=np.float64)
    v = np.ascontiguousarray(values, dtype=np.float64)
    d = np.ascontiguousarray(dones, dtype=np.float64)
    b = np.ascontiguousarray(bootstrap, dtype=np.float64)
    T = r.shape[0]
    N = r.size // max(T, 1)
    adv, ret = np.zeros_like(r), np.zeros_like(r)
    _lib().orc_gae(ctypes.c_int64(T), ctypes.c_int64(N), _vp(r), _vp(v), _vp(d), _vp(b),
                   ctypes.c_double(gamma), ctypes.c_double(lam), _vp(adv), _vp(ret))
    return adv, ret


def norm_update(count, mean, var, batch):
    x = np.ascontiguousarray(np.atleast_2d(batch), dtype=np.float64)
    m = np.array(mean, dtype=np.float64)
    v = np.array(var, dtype=np.float64)
    c = ctypes.c_double(count)
    _lib().orc_norm_update(ctypes.c_int64(x.shape[0]), x.shape[1], _vp(x), ctypes.byref(c),
                           _vp(m), _vp(v))
    return c.value, m, v


def norm_apply(count, mean, var, eps, batch, invert=False):
    x = np.ascontiguousarray(batch, dtype=np.float64)
    D = x.shape[-1]
    m = np.ascontiguousarray(mean, dtype=np.float64)
    v = np.ascontiguousarray(var, dtype=np.float64)
    out = np.zeros_like(x)
    _lib().orc_norm_apply(ctypes.c_int64(x.size // D), D, _vp(x), ctypes.c_double(count), _vp(m),
                          _vp(v), ctypes.c_double(eps), int(invert), _vp(out))
    return out


def pixel_normalize(img):
    """ppo.pixel_normalize on [n, h, w, c]: float64 [n, h, w, c]."""
    x = np.ascontiguousarray(img, dtype=np.float64)
    n, h, w, c = x.shape
    out = np.zeros_like(x)
    _lib().orc_pixel_normalize(ctypes.c_int64(n), ctypes.c_int64(h * w), c, _vp(x), _vp(out))
    return out
