"""Synthetic rollout workloads of BASELINE.md §2 (shared by bench.py and tests).

Host-side numpy generation (numpy.random.default_rng(seed)); behaviour
log-probs and values are filled by whoever owns the networks (the GPU arm
with its own kernels, the CPU reference arm with the reference/oracle).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

CONFIGS = {
    # name: (T, N, obs, critic_obs, act, hidden)
    "cfg1": (24, 1024, 48, 48, 12, (256, 128, 128)),
    "cfg2": (24, 4096, 235, 235, 12, (512, 256, 128)),
    "cfg5": (24, 16384, 98, 101, 29, (512, 256, 128)),
}


@dataclass
class HostRollout:
    T: int
    N: int
    obs: np.ndarray
    critic_obs: np.ndarray
    actions: np.ndarray
    rewards: np.ndarray
    terminated: np.ndarray
    truncated: np.ndarray
    bootstrap_value: np.ndarray
    truncation_values: np.ndarray
    behavior_log_prob: np.ndarray = None
    values: np.ndarray = None


def make_rollout(name: str, seed: int = 0, alloc=np.empty) -> HostRollout:
    """obs/critic_obs/actions ~ N(0,1) f32; rewards 0.1 N(0,1); terminated
    Bernoulli(0.01); truncated Bernoulli(0.005) & ~terminated; bootstrap N(0,1);
    truncation_values N(0,1)*truncated.  ``alloc`` may return pinned arrays."""
    T, N, od, cd, ad, _ = CONFIGS[name]
    rng = np.random.default_rng(seed)

    def fill(shape, dtype, values):
        out = alloc(shape, dtype)
        out[...] = values
        return out

    obs = fill((T, N, od), np.float32, rng.standard_normal((T, N, od), dtype=np.float32))
    cobs = fill((T, N, cd), np.float32, rng.standard_normal((T, N, cd), dtype=np.float32))
    act = fill((T, N, ad), np.float32, rng.standard_normal((T, N, ad), dtype=np.float32))
    rew = 0.1 * rng.normal(size=(T, N))
    term = rng.random((T, N)) < 0.01
    trunc = (rng.random((T, N)) < 0.005) & ~term
    boot = rng.normal(size=N)
    tv = rng.normal(size=(T, N)) * trunc
    return HostRollout(T, N, obs, cobs, act, rew, term, trunc, boot, tv)
