"""GAE / V-trace and the FlashSAC collector transforms on the device
(mirror of R:algos/estimators.py).

``gae`` and ``vtrace`` keep the reference signatures and return device
float32 [T, N] tensors computed by ul_gae_f32 / ul_vtrace_f32 (float64
arithmetic inside the kernel).  ``ReturnStdNormalizer`` / ``NStepPacker`` /
``nstep_and_reward_norm`` keep the reference API over the n-step kernels of
csrc/nstep.cu.
"""

from __future__ import annotations

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


# ------------------------------------------- collector-side transforms
# R:algos/estimators.py:125-224 run per env in Python on the reference's
# collector thread.  Here the same objects drive the device kernels of
# csrc/nstep.cu (replaypath.DeviceNStepReplay): the pending n-step windows,
# the discounted-return statistics and the packing live in HBM; push()
# returns the emitted transitions as the reference's tuples (one D2H of the
# emitted rows) so a host collector can keep its code unchanged -- or use
# DeviceNStepReplay directly and never bring the rows back.
class ReturnStdNormalizer:
    """Running std of per-env discounted returns (R:algos/estimators.py:125-163).
    The statistics live on the device; they are bound into an NStepPacker by
    ``nstep_and_reward_norm`` (fused normalise + pack), or driven alone by
    ``normalize`` (a 1-step packer over the rewards)."""

    def __init__(self, gamma: float, g_max: float, n_envs: int, eps: float = 1e-8):
        self.gamma, self.g_max, self.n_envs, self.eps = float(gamma), float(g_max), int(n_envs), eps
        self._engine = None  # the DeviceNStepReplay holding the statistics

    def _stats(self):
        if self._engine is None:
            return (0.0, 0.0, 0.0, 1.0)
        return self._engine.norm_stats()

    @property
    def count(self) -> float:
        return self._stats()[0]

    @property
    def mean(self) -> float:
        return self._stats()[1]

    @property
    def m2(self) -> float:
        return self._stats()[2]

    @property
    def std(self) -> float:
        return self._stats()[3]

    def normalize(self, rewards, done):
        """Update the return statistics with this step and return the clipped
        normalised rewards (R:algos/estimators.py:153-163)."""
        from ..replaypath.device_insert import DeviceNStepReplay

        if self._engine is None:
            self._engine = DeviceNStepReplay(1, self.gamma, self.n_envs, 1, 1,
                                             capacity=self.n_envs, norm_gamma=self.gamma,
                                             g_max=self.g_max, eps=self.eps)
        elif self._engine.n != 1:
            raise RuntimeError("normaliser is bound to an NStepPacker; use nstep_and_reward_norm")
        z = np.zeros((self.n_envs, 1), np.float32)
        done = np.asarray(done, bool)
        eng = self._engine
        h0 = eng.head
        eng.push(z, z, np.asarray(rewards, np.float64), z, done, np.zeros_like(done))
        rows = eng.rows(h0, eng.head)
        return rows[:, 2].astype(np.float64)  # RowCodec(1, 1): obs | act | reward | ...


class NStepPacker:
    """Per-env n-step packing (R:algos/estimators.py:166-207) on the device."""

    def __init__(self, n: int, gamma: float, n_envs: int):
        if n < 1:
            raise ValueError("n must be >= 1")
        self.n, self.gamma, self.n_envs = int(n), float(gamma), int(n_envs)
        self._engine = None
        self._norm = None

    def _bind(self, obs_dim: int, act_dim: int, norm=None):
        from ..replaypath.device_insert import DeviceNStepReplay

        if self._engine is None:
            if norm is not None and norm._engine is not None:
                raise RuntimeError("normaliser already driven on its own")
            self._engine = DeviceNStepReplay(
                self.n, self.gamma, self.n_envs, obs_dim, act_dim,
                capacity=self.n_envs * (self.n + 1),
                norm_gamma=norm.gamma if norm is not None else None,
                g_max=norm.g_max if norm is not None else 10.0,
                eps=norm.eps if norm is not None else 1e-8)
            self._norm = norm
            if norm is not None:
                norm._engine = self._engine
        elif norm is not self._norm:
            raise RuntimeError("an NStepPacker is bound to one normaliser (or none)")
        return self._engine

    def push(self, obs, actions, rewards, next_obs, terminated, truncated, _norm=None):
        """One env step; returns the emitted (obs, action, reward, next_obs,
        terminated, n_used) tuples in the reference's env-major order."""
        obs = np.asarray(_dev.to_numpy(obs), np.float32)
        actions = np.asarray(_dev.to_numpy(actions), np.float32)
        eng = self._bind(obs.shape[1], actions.shape[1], _norm)
        h0 = eng.head
        eng.push(obs, actions, np.asarray(_dev.to_numpy(rewards), np.float64), next_obs,
                 terminated, truncated)
        if eng.head == h0:
            return []
        rows = eng.rows(h0, eng.head)
        d, a = eng.obs_dim, eng.act_dim
        return [(r[:d].copy(), r[d:d + a].copy(), float(r[d + a]), r[d + a + 1:2 * d + a + 1].copy(),
                 bool(r[2 * d + a + 1] > 0.5), int(r[2 * d + a + 2])) for r in rows]


def nstep_and_reward_norm(packer, norm, obs, actions, rewards, next_obs, terminated, truncated):
    """Reward normalisation (optional) + n-step packing of one step
    (R:algos/estimators.py:210-224), fused on the device."""
    return packer.push(obs, actions, rewards, next_obs, terminated, truncated, _norm=norm)
