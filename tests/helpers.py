"""Shared synthetic-rollout builders for the GPU tests (oracle nets fill
values / behaviour log-probs, BASELINE.md §2 recipe)."""

import numpy as np

from oracle import port as O


def _synthetic(T, N, od, cd, ad, hid, seed=0):
    """BASELINE.md synthetic recipe (values / blogp from the oracle nets)."""
    rng = np.random.default_rng(seed)
    actor = O.net_init((od, *hid, ad), 0)
    critic = O.net_init((cd, *hid, 1), 1)
    obs = rng.normal(size=(T, N, od)).astype(np.float32)
    cobs = rng.normal(size=(T, N, cd)).astype(np.float32)
    act = rng.normal(size=(T, N, ad)).astype(np.float32)
    rew = 0.1 * rng.normal(size=(T, N))
    term = rng.random((T, N)) < 0.01
    trunc = (rng.random((T, N)) < 0.005) & ~term
    boot = rng.normal(size=N)
    tv = rng.normal(size=(T, N)) * trunc
    mean, _ = O.mlp_forward(actor, obs.reshape(-1, od))
    blogp = O.gauss_logp(mean, actor.log_std, act.reshape(-1, ad)).reshape(T, N).astype(np.float64)
    vals = O.value_forward(critic, cobs.reshape(-1, cd))[0].reshape(T, N).astype(np.float64)
    seg = dict(obs=obs, critic_obs=cobs, actions=act, behavior_log_prob=blogp, rewards=rew,
               terminated=term, truncated=trunc, values=vals, bootstrap_value=boot,
               truncation_values=tv)
    return seg, actor, critic
