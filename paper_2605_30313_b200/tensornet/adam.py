"""Adam with bias correction and global-norm clipping (mirror of R:tensornet/adam.py).

The host OptState keeps the reference fields (m, v, t, lr, betas, eps); m and
v are device Grads records.  Each call uploads a small ul_opt_ctl record,
runs ul_adam_step / ul_clip_global_norm and reads the control header back so
that DivergenceError is raised synchronously, exactly where the reference
raises it (R:tensornet/adam.py:55-56).  The PPO/APPO/SAC update plans keep this
record device-resident instead and never round-trip per step.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from .. import _dev, _lib
from ..errors import DivergenceError
from .mlp import Grads, ModelParams

_HDR = _lib.OptCtl.part.offset  # bytes of the control header (without partials)


@dataclass
class OptState:
    """R:tensornet/adam.py:16-27."""

    m: Grads
    v: Grads
    t: int = 0
    lr: float = 1e-3
    betas: tuple = (0.9, 0.999)
    eps: float = 1e-8

    @classmethod
    def for_params(cls, params: ModelParams, lr: float) -> "OptState":
        return cls(m=Grads.zeros_like(params), v=Grads.zeros_like(params), lr=lr)


class _Ctl:
    """A device ul_opt_ctl plus its host mirror."""

    def __init__(self, lrs, ts, betas, eps, max_norm):
        self.host = _lib.OptCtl()
        lr_arr = (C.c_double * len(lrs))(*lrs)
        _lib.call("ul_opt_ctl_init", C.byref(self.host), len(lrs), lr_arr, betas[0], betas[1],
                  eps, max_norm)
        for i, t in enumerate(ts):
            self.host.t[i] = int(t)
        self.dev = _dev.zeros(C.sizeof(_lib.OptCtl), dtype=torch.uint8, device="cuda")
        _lib.call("ul_memcpy_async", _dev.ptr(self.dev), C.addressof(self.host), _HDR,
                  _dev.stream())

    def read(self) -> _lib.OptCtl:
        _lib.call("ul_memcpy_async", C.addressof(self.host), _dev.ptr(self.dev), _HDR,
                  _dev.stream())
        _lib.call("ul_stream_sync", _dev.stream())
        return self.host


def _seg(records):
    bufs = [r.buf for r in records]
    return _lib.ptr_array([_dev.ptr(b) for b in bufs]), _lib.i64_array([b.numel() for b in bufs])


def clip_global_norm(grads_list, max_norm: float) -> float:
    """Scale all grads in place so their joint norm <= max_norm; returns the
    pre-clip norm (R:tensornet/adam.py:30-40)."""
    grads_list = list(grads_list)
    if not grads_list:
        return 0.0
    _dev.require_cuda()
    out = 0.0
    # the kernel handles UL_MAX_SEG segments jointly; larger lists fold in chunks
    if len(grads_list) > _lib.UL_MAX_SEG:
        total = float(np.sqrt(sum(clip_global_norm([g], 0.0) ** 2 for g in grads_list)))
        if max_norm > 0 and total > max_norm:
            f = max_norm / (total + 1e-12)
            for g in grads_list:
                g.scale_(f)
        return total
    ctl = _Ctl([0.0] * len(grads_list), [0] * len(grads_list), (0.9, 0.999), 1e-8, max_norm)
    g, n = _seg(grads_list)
    _lib.call("ul_clip_global_norm", g, n, len(grads_list), _dev.ptr(ctl.dev), _dev.stream())
    out = float(ctl.read().norm)
    return out


def adam_step(params: ModelParams, grads: Grads, opt: OptState, max_grad_norm: float = 0.0):
    """One textbook Adam step on the device; mutates and returns (params, opt)
    (R:tensornet/adam.py:43-80).  Non-finite gradients raise DivergenceError
    and leave params / opt untouched."""
    _dev.require_cuda()
    ctl = _Ctl([opt.lr], [opt.t], opt.betas, opt.eps, max_grad_norm)
    _lib.call("ul_adam_step", _lib.ptr_array([_dev.ptr(params.buf)]),
              _lib.ptr_array([_dev.ptr(grads.buf)]), _lib.ptr_array([_dev.ptr(opt.m.buf)]),
              _lib.ptr_array([_dev.ptr(opt.v.buf)]), _lib.i64_array([params.buf.numel()]), 1,
              _dev.ptr(ctl.dev), 1, _dev.stream())
    h = ctl.read()
    if h.seg_bad[0]:
        raise DivergenceError("non-finite gradients in adam_step")
    opt.t = int(h.t[0])
    return params, opt
