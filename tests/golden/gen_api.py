"""Golden vectors of the per-call SAC / Gaussian-head API, produced by running
the UNMODIFIED reference:

  R:tensornet/distributions.py  gaussian_dist (4 modes), squashed_log_prob,
                                sample_squashed
  R:algos/sac.py                critic_target, critic_loss_and_grads,
                                actor_loss_and_grads, alpha_loss_and_grad

    python tests/golden/gen_api.py      (build container, /root/reference present)
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

from unilite.algos import (SacConfig, SacState, actor_loss_and_grads,  # noqa: E402
                           alpha_loss_and_grad, critic_loss_and_grads, critic_target)
from unilite.envcore.rng import stream  # noqa: E402
from unilite.tensornet import (Arch, gaussian_dist, init_params, sample_squashed,  # noqa: E402
                               squashed_log_prob)


def main():
    rng = np.random.default_rng(11)
    out = {}
    # ---- Gaussian heads
    n, A = 300, 7
    mean = rng.normal(size=(n, A))
    log_std = rng.normal(scale=0.3, size=A)
    act = np.tanh(rng.normal(size=(n, A)))
    out["g_mean"], out["g_log_std"], out["g_act"] = mean, log_std, act
    for mode, (action, squashed) in enumerate(((None, False), (act, False), (None, True),
                                               (act, True))):
        r = stream(4, f"dist{mode}")
        s, lp, ent = gaussian_dist(mean, log_std, action=action, squashed=squashed, rng=r)
        out[f"g{mode}_sample"], out[f"g{mode}_logp"], out[f"g{mode}_ent"] = s, lp, ent
    u = rng.normal(size=(n, A))
    out["g_u"] = u
    out["g_sqlp"] = squashed_log_prob(mean, log_std, u, np.tanh(u))
    m32 = mean.astype(np.float32)
    ls32 = log_std.astype(np.float32)
    eps32 = rng.normal(size=(n, A)).astype(np.float32)
    a, uu, lp = sample_squashed(m32, ls32, eps32)
    out["s_eps"], out["s_a"], out["s_u"], out["s_logp"] = eps32, a, uu, lp
    # ---- SAC building blocks (obs 11, act 4, 64-32 nets, batch 257)
    od, ad, B = 11, 4, 257
    cfg = SacConfig()
    actor = init_params(Arch(od, (64, 32), ad), 0)
    q1 = init_params(Arch(od + ad, (64, 32), 1), 1)
    q2 = init_params(Arch(od + ad, (64, 32), 1), 2)
    st = SacState.create(actor, q1, q2, cfg)
    p = st.params
    p.log_alpha = float(np.log(0.2))
    # targets != online critics
    for (w, b) in p.q1_targ.layers:
        w += rng.normal(scale=0.05, size=w.shape).astype(np.float32)
    batch = dict(obs=rng.normal(size=(B, od)).astype(np.float32),
                 action=np.tanh(rng.normal(size=(B, ad))).astype(np.float32),
                 reward=rng.normal(size=B).astype(np.float32),
                 next_obs=rng.normal(size=(B, od)).astype(np.float32),
                 terminated=rng.random(B) < 0.1, n_used=rng.integers(1, 4, B))
    for k, v in batch.items():
        out[f"b_{k}"] = v
    out["p_actor"], out["p_q1"], out["p_q2"] = actor.flat(), q1.flat(), q2.flat()
    out["p_q1t"], out["p_q2t"] = p.q1_targ.flat(), p.q2_targ.flat()
    out["p_log_alpha"] = np.array(p.log_alpha)
    y = critic_target(p, batch, cfg.gamma, stream(1, "learner"))
    out["y"] = y
    q_in = np.concatenate([batch["obs"], batch["action"]], axis=-1)
    loss, g, qp = critic_loss_and_grads(p.q1, q_in, y)
    out["c_loss"], out["c_grads"], out["c_pred"] = np.array(loss), g.flat(), qp
    eps = stream(1, "actor").standard_normal((B, ad))
    out["a_eps"] = eps
    aloss, ag, logp = actor_loss_and_grads(p, batch["obs"], eps)
    out["a_loss"], out["a_grads"], out["a_logp"] = np.array(aloss), ag.flat(), logp
    al, dla = alpha_loss_and_grad(p.log_alpha, logp, -1.5)
    out["al"] = np.array([al, dla])
    np.savez_compressed(OUT / "api.npz", **out)
    print("wrote", OUT / "api.npz")


if __name__ == "__main__":
    main()
