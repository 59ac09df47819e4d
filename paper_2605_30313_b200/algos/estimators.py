"""GAE / V-trace on the device + the host collector-side packers
(mirror of R:algos/estimators.py).

``gae`` and ``vtrace`` keep the reference signatures and return device
float32 [T, N] tensors computed by ul_gae_f32 / ul_vtrace_f32 (float64
arithmetic inside the kernel).  ``ReturnStdNormalizer`` and ``NStepPacker``
run on the collector thread in the reference (R:runtime/sac_runner.py:220-247)
and stay host code here.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .. import _dev, _lib


def _as_dev(x, dtype=torch.float32) -> torch.Tensor:
    if isinstance(x, torch.Tensor) and x.is_cuda:
        return x if x.dtype == dtype and x.is_contiguous() else x.to(dtype).contiguous()
    npd = np.uint8 if dtype == torch.uint8 else np.float32
    a = np.ascontiguousarray(np.asarray(x), dtype=npd)
    out = torch.empty(a.shape, dtype=dtype, device="cuda")
    _dev.h2d(out, a)
    return out


def _shape(x):
    return tuple(x.shape) if hasattr(x, "shape") else np.asarray(x).shape


def gae(rewards, values, terminated, truncated, bootstrap_value, gamma: float, lam: float,
        truncation_values=None):
    """Generalized advantage estimation over a (T, B) rollout (R:algos/estimators.py:29-63)."""
    _dev.require_cuda()
    if not (_shape(rewards) == _shape(values) == _shape(terminated) == _shape(truncated)):
        raise ValueError("rewards/values/terminated/truncated must share (T, B)")
    shape = _shape(rewards)
    if len(shape) != 2:
        raise ValueError("rollout arrays must be (T, B)")
    T, N = shape
    r, v = _as_dev(rewards), _as_dev(values)
    te, tr = _as_dev(terminated, torch.uint8), _as_dev(truncated, torch.uint8)
    boot = _as_dev(bootstrap_value)
    tv = None if truncation_values is None else _as_dev(truncation_values)
    adv = torch.empty((T, N), dtype=torch.float32, device=r.device)
    ret = torch.empty_like(adv)
    _lib.call("ul_gae_f32", _dev.ptr(r), _dev.ptr(v), _dev.ptr(te), _dev.ptr(tr), _dev.ptr(tv),
              _dev.ptr(boot), T, N, float(gamma), float(lam), _dev.ptr(adv), _dev.ptr(ret),
              _dev.stream())
    return adv, ret


def vtrace(behavior_log_prob, target_log_prob, rewards, values, terminated, bootstrap_value,
           gamma: float, rho_bar: float, c_bar: float, truncated=None, truncation_values=None):
    """Clipped-IS value targets and PG advantages (R:algos/estimators.py:66-122)."""
    _dev.require_cuda()
    shp = _shape(rewards)
    if not (shp == _shape(values) == _shape(terminated) == _shape(behavior_log_prob)
            == _shape(target_log_prob)):
        raise ValueError("vtrace inputs must share (T, B)")
    T, N = shp
    bl, tl = _as_dev(behavior_log_prob), _as_dev(target_log_prob)
    r, v = _as_dev(rewards), _as_dev(values)
    te = _as_dev(terminated, torch.uint8)
    tr = None if truncated is None else _as_dev(truncated, torch.uint8)
    tv = None if truncation_values is None else _as_dev(truncation_values)
    boot = _as_dev(bootstrap_value)
    vs = torch.empty((T, N), dtype=torch.float32, device=r.device)
    pg = torch.empty_like(vs)
    _lib.call("ul_vtrace_f32", _dev.ptr(bl), _dev.ptr(tl), _dev.ptr(r), _dev.ptr(v), _dev.ptr(te),
              _dev.ptr(tr), _dev.ptr(tv), _dev.ptr(boot), T, N, float(gamma), float(rho_bar),
              float(c_bar), _dev.ptr(vs), _dev.ptr(pg), _dev.stream())
    return vs, pg


# ------------------------------------------------------- host collector side
@dataclass
class ReturnStdNormalizer:
    """Running std of per-env discounted returns (R:algos/estimators.py:125-163).
    Host-side: it runs on the collector thread before replay insertion."""

    gamma: float
    g_max: float
    n_envs: int
    eps: float = 1e-8
    returns: np.ndarray = None
    count: float = 0.0
    mean: float = 0.0
    m2: float = 0.0

    def __post_init__(self) -> None:
        if self.returns is None:
            self.returns = np.zeros(self.n_envs, dtype=np.float64)

    @property
    def std(self) -> float:
        return 1.0 if self.count < 2 else float(np.sqrt(self.m2 / self.count))

    def normalize(self, rewards, done):
        rewards = np.asarray(rewards, dtype=np.float64)
        self.returns = self.returns * self.gamma * (~np.asarray(done, bool)) + rewards
        # sequential Welford over the envs, same order as the reference loop
        for g in self.returns:
            self.count += 1
            d = g - self.mean
            self.mean += d / self.count
            self.m2 += d * (g - self.mean)
        bound = (1.0 - self.gamma) * self.g_max
        return np.clip(rewards / (self.std + self.eps), -bound, bound)


class NStepPacker:
    """Per-env n-step packing (R:algos/estimators.py:166-207); host-side."""

    def __init__(self, n: int, gamma: float, n_envs: int):
        if n < 1:
            raise ValueError("n must be >= 1")
        self.n, self.gamma = n, gamma
        self._pending = [[] for _ in range(n_envs)]

    def push(self, obs, actions, rewards, next_obs, terminated, truncated):
        out = []
        done = np.asarray(terminated, bool) | np.asarray(truncated, bool)
        for e, pend in enumerate(self._pending):
            for item in pend:
                item[2] += (self.gamma ** item[3]) * rewards[e]
                item[3] += 1
            pend.append([obs[e].copy(), actions[e].copy(), float(rewards[e]), 1])
            if done[e]:
                out.extend((it[0], it[1], it[2], next_obs[e].copy(), bool(terminated[e]), it[3])
                           for it in pend)
                pend.clear()
            elif pend[0][3] == self.n:
                it = pend.pop(0)
                out.append((it[0], it[1], it[2], next_obs[e].copy(), False, self.n))
        return out


def nstep_and_reward_norm(packer, norm, obs, actions, rewards, next_obs, terminated, truncated):
    """R:algos/estimators.py:210-224."""
    if norm is not None:
        done = np.asarray(terminated, bool) | np.asarray(truncated, bool)
        rewards = norm.normalize(rewards, done)
    return packer.push(obs, actions, rewards, next_obs, terminated, truncated)
