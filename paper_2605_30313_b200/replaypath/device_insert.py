"""FlashSAC collector transforms + replay insert on the device (SURVEY.md
8(f) item 3): the per-env Python loops of ReturnStdNormalizer.normalize
(R:algos/estimators.py:153-163) and NStepPacker.push (:166-207), run before
replay insertion in R:runtime/sac_runner.py:220-247, become four kernels
(csrc/nstep.cu) that write packed RowCodec rows straight into an HBM replay
ring; sampling reads that ring with the K6 gather (``DeviceRows``)."""

from __future__ import annotations

import numpy as np
import torch

from .. import _dev, _lib


def _dev_arr(x, dtype) -> torch.Tensor:
    if isinstance(x, torch.Tensor) and x.is_cuda:
        return x.to(dtype).contiguous()
    npd = np.uint8 if dtype == torch.uint8 else np.float32
    a = np.ascontiguousarray(np.asarray(x), dtype=npd)
    t = torch.empty(a.shape, dtype=dtype, device="cuda")
    _dev.h2d(t, a)
    return t


class DeviceNStepReplay:
    """n-step packer (+ optional return-std reward normaliser) feeding an HBM
    replay ring of ``capacity`` codec rows.  ``push`` takes one environment
    step of all envs; rows are inserted in the reference's order."""

    def __init__(self, n: int, gamma: float, n_envs: int, obs_dim: int, act_dim: int,
                 capacity: int, norm_gamma: float | None = None, g_max: float = 10.0,
                 eps: float = 1e-8):
        if n < 1:
            raise ValueError("n must be >= 1")
        _dev.require_cuda()
        self.n, self.gamma, self.n_envs = n, gamma, n_envs
        self.obs_dim, self.act_dim, self.capacity = obs_dim, act_dim, capacity
        self.norm_gamma, self.g_max, self.eps = norm_gamma, g_max, eps
        nb = _lib.lib().ul_nstep_state_bytes(n_envs, n, obs_dim, act_dim)
        self.state = _dev.zeros(nb, dtype=torch.uint8, device="cuda")
        self.width = 2 * obs_dim + act_dim + 3
        self.ldr = (self.width + 3) // 4 * 4
        self.ring = _dev.zeros((capacity, self.ldr), dtype=torch.float32, device="cuda")
        self.head = 0  # absolute rows inserted
        self._count = _dev.pinned_empty((1,), np.int64)

    def push(self, obs, actions, rewards, next_obs, terminated, truncated) -> int:
        """nstep_and_reward_norm + insert for one step (R:algos/estimators.py:210-224);
        returns the number of rows inserted."""
        o = _dev_arr(obs, torch.float32)
        a = _dev_arr(actions, torch.float32)
        r = _dev_arr(rewards, torch.float32)
        no = _dev_arr(next_obs, torch.float32)
        te = _dev_arr(terminated, torch.uint8)
        tr = _dev_arr(truncated, torch.uint8)
        s = _dev.stream()
        _lib.call("ul_nstep_push", _dev.ptr(self.state), self.n_envs, self.n, self.obs_dim,
                  self.act_dim, float(self.gamma),
                  float(self.norm_gamma) if self.norm_gamma else 0.0, float(self.g_max),
                  float(self.eps), _dev.ptr(o), _dev.ptr(a), _dev.ptr(r), _dev.ptr(no),
                  _dev.ptr(te), _dev.ptr(tr), _dev.ptr(self.ring), self.capacity, self.ldr,
                  self.head, self._count.ctypes.data, s)
        _lib.call("ul_stream_sync", s)
        k = int(self._count[0])
        self.head += k
        return k

    def norm_stats(self) -> tuple:
        out = _dev.pinned_empty((4,), np.float64)
        s = _dev.stream()
        _lib.call("ul_nstep_norm_stats", _dev.ptr(self.state), self.n_envs, self.n,
                  self.obs_dim, self.act_dim, out.ctypes.data, s)
        _lib.call("ul_stream_sync", s)
        return tuple(float(x) for x in out)

    def rows(self, lo: int, hi: int) -> np.ndarray:
        """Codec rows of absolute indices [lo, hi) (host copy, for checks)."""
        idx = np.arange(lo, hi) % self.capacity
        return self.ring[torch.as_tensor(idx, device="cuda")][:, :self.width].cpu().numpy()

    def sample(self, indices):
        """A DeviceRows batch of absolute indices for sac_update (window-checked)."""
        from ..algos.sac import DeviceRows

        idx = torch.as_tensor(np.asarray(indices, np.int64), device="cuda")
        lo = max(0, self.head - self.capacity)
        return DeviceRows(self.ring, self.ldr, idx, len(indices), modulo=self.capacity, lo=lo,
                          hi=self.head)
