"""Diagonal Gaussian heads on the device (mirror of R:tensornet/distributions.py)."""

from __future__ import annotations

import numpy as np
import torch

from .. import _dev, _lib

LOG_2PI = float(np.log(2.0 * np.pi))


def gaussian_log_prob(mean, log_std, action) -> torch.Tensor:
    """log N(action; mean, exp(log_std)) summed over action dims
    (R:tensornet/distributions.py:11-18), kernel ul_gaussian_logp."""
    m = _dev.to_device_f32(mean)
    a = _dev.to_device_f32(action)
    ls = _dev.to_device_f32(np.asarray(_dev.to_numpy(log_std), np.float32).reshape(1, -1))
    if m.dim() != 2 or tuple(m.shape) != tuple(a.shape):
        raise ValueError("mean/action must be (B, A) and agree")
    out = torch.empty(m.shape[0], dtype=torch.float32, device=m.device)
    _lib.call("ul_gaussian_logp", _dev.ptr(m), m.stride(0), _dev.ptr(ls), _dev.ptr(a), a.stride(0),
              m.shape[0], m.shape[1], _dev.ptr(out), _dev.stream())
    return out


def gaussian_entropy(log_std, batch: int | None = None):
    """sum(log_std + 0.5 (ln 2pi + 1)) (R:tensornet/distributions.py:21-26);
    a host scalar (it depends only on the A log-std values)."""
    ls = np.asarray(_dev.to_numpy(log_std))
    h = float(np.sum(ls + 0.5 * (LOG_2PI + 1.0)))
    return np.float64(h) if batch is None else np.full(batch, h)
