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


def _mean_logstd_f64(mean, log_std):
    m = _dev.to_device_f64(mean)
    if m.dim() == 1:
        m = m.reshape(1, -1)
    ls = _dev.to_device_f64(np.asarray(_dev.to_numpy(log_std), np.float64).reshape(-1))
    if m.dim() != 2 or m.shape[1] != ls.numel():
        raise ValueError("mean must be (B, A) with A log-std entries")
    return m, ls


def gaussian_dist(mean, log_std, action=None, squashed: bool = False, rng=None):
    """Sample (or evaluate) a diagonal Gaussian head (R:tensornet/distributions.py:29-63):
    (sample, log_prob, entropy), float64 like the reference.  The standard
    normals of a sample come from `rng` (the reference draw), the density and
    the tanh squash run in ul_gaussian_dist."""
    m, ls = _mean_logstd_f64(mean, log_std)
    n, A = m.shape
    entropy = gaussian_entropy(_dev.to_numpy(ls), batch=n)
    if action is None:
        if rng is None:
            raise ValueError("sampling requires an rng")
        x = _dev.to_device_f64(rng.standard_normal((n, A)))
        mode = 2 if squashed else 0
    else:
        x = _dev.to_device_f64(np.atleast_2d(_dev.to_numpy(action)))
        if tuple(x.shape) != (n, A):
            raise ValueError("action must match mean's shape")
        mode = 3 if squashed else 1
    sample = torch.empty((n, A), dtype=torch.float64, device=m.device)
    logp = torch.empty(n, dtype=torch.float64, device=m.device)
    _lib.call("ul_gaussian_dist", _dev.ptr(m), A, _dev.ptr(ls), _dev.ptr(x), A, None, n, A, mode,
              _dev.ptr(sample), None, _dev.ptr(logp), _dev.stream())
    return sample, logp, entropy


def squashed_log_prob(mean, log_std, u, a) -> torch.Tensor:
    """log-density of a = tanh(u), u ~ N(mean, exp(log_std))
    (R:tensornet/distributions.py:66-70), float64."""
    m, ls = _mean_logstd_f64(mean, log_std)
    n, A = m.shape
    ud, ad = _dev.to_device_f64(u).reshape(n, A), _dev.to_device_f64(a).reshape(n, A)
    logp = torch.empty(n, dtype=torch.float64, device=m.device)
    _lib.call("ul_gaussian_dist", _dev.ptr(m), A, _dev.ptr(ls), _dev.ptr(ud), A, _dev.ptr(ad),
              n, A, 4, None, None, _dev.ptr(logp), _dev.stream())
    return logp


def sample_squashed(mean, log_std, eps) -> tuple:
    """Reparameterized squashed sample from fixed noise
    (R:tensornet/distributions.py:73-84): (a, u, log_prob), float32 like the
    reference's float32 heads."""
    m = _dev.to_device_f32(mean)
    e = _dev.to_device_f32(eps)
    ls = _dev.to_device_f32(np.asarray(_dev.to_numpy(log_std), np.float32).reshape(1, -1))
    if m.dim() != 2 or tuple(m.shape) != tuple(e.shape):
        raise ValueError("mean/eps must be (B, A) and agree")
    n, A = m.shape
    a = torch.empty((n, A), dtype=torch.float32, device=m.device)
    u = torch.empty_like(a)
    logp = torch.empty(n, dtype=torch.float32, device=m.device)
    _lib.call("ul_sample_squashed", _dev.ptr(m), m.stride(0), _dev.ptr(ls), _dev.ptr(e),
              e.stride(0), n, A, _dev.ptr(a), _dev.ptr(u), _dev.ptr(logp), _dev.stream())
    return a, u, logp
