"""Running observation normaliser on the device (mirror of R:tensornet/normalizer.py).

Statistics live in a float64 HBM vector [count, mean[D], var[D]]; update and
apply are the ul_norm_update / ul_norm_apply kernels (K3).  ``count`` / ``mean``
/ ``var`` properties read the statistics back to the host (D2H).
"""

from __future__ import annotations

import numpy as np
import torch

from .. import _dev, _lib

CLIP = 10.0
EPS = 1e-8


class Normalizer:
    def __init__(self, dim: int, count: float = 0.0, mean=None, var=None, frozen: bool = False):
        _dev.require_cuda()
        self.dim = int(dim)
        self.frozen = bool(frozen)
        host = np.zeros(1 + 2 * self.dim)
        host[0] = count
        if mean is not None:
            host[1:1 + self.dim] = np.asarray(mean, np.float64)
        if var is not None:
            host[1 + self.dim:] = np.asarray(var, np.float64)
        self.state = torch.empty(host.size, dtype=torch.float64, device="cuda")
        _dev.h2d(self.state, host)
        self.work = _dev.zeros(_lib.lib().ul_norm_work_bytes(self.dim), dtype=torch.uint8,
                                device="cuda")

    # host views (D2H)
    @property
    def count(self) -> float:
        return float(_dev.to_numpy(self.state[:1])[0])

    @property
    def mean(self) -> np.ndarray:
        return _dev.to_numpy(self.state[1:1 + self.dim]).copy()

    @property
    def var(self) -> np.ndarray:
        return _dev.to_numpy(self.state[1 + self.dim:]).copy()

    def _dev_batch(self, batch) -> torch.Tensor:
        x = _dev.to_device_f32(batch) if not (isinstance(batch, torch.Tensor) and batch.is_cuda
                                            and batch.dtype == torch.float32
                                            and batch.stride(-1) == 1) else batch
        if x.dim() != 2 or x.shape[1] != self.dim:
            raise ValueError(f"batch dim {tuple(x.shape)} != normalizer dim {self.dim}")
        return x

    def update(self, batch) -> None:
        """Parallel-Welford merge of a batch (R:tensornet/normalizer.py:27-45)."""
        if self.frozen:
            return
        x = self._dev_batch(batch)
        _lib.call("ul_norm_update", _dev.ptr(x), x.shape[0], self.dim, x.stride(0),
                  _dev.ptr(self.state), _dev.ptr(self.work), 0, _dev.stream())

    def apply(self, batch) -> torch.Tensor:
        """clip((x - mean)/sqrt(var + 1e-8), +-10) as float32 (:47-49)."""
        x = self._dev_batch(batch)
        out = torch.empty((x.shape[0], self.dim), dtype=torch.float32, device=x.device)
        _lib.call("ul_norm_apply", _dev.ptr(x), x.shape[0], self.dim, x.stride(0),
                  _dev.ptr(self.state), _dev.ptr(out), self.dim, _dev.stream())
        return out

    def unapply(self, batch) -> np.ndarray:
        return _dev.to_numpy(batch) * np.sqrt(self.var + EPS) + self.mean

    def copy(self) -> "Normalizer":
        return Normalizer(self.dim, self.count, self.mean, self.var, self.frozen)


def norm_update_apply(norm: Normalizer, batch) -> torch.Tensor:
    """R:tensornet/normalizer.py:61-66."""
    shape = tuple(batch.shape)
    if shape[-1] != norm.dim:
        raise ValueError(f"batch dim {shape[-1]} != normalizer dim {norm.dim}")
    norm.update(batch)
    return norm.apply(batch)
