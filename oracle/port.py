"""Numpy restatement of the reference learner hot path (TEST INFRASTRUCTURE).

Every function names the reference lines it restates; ``R:`` is
``/root/reference/pkg/src/unilite/``.  The restatement keeps the reference's
dtype flow (Appendix B of SURVEY.md): float32 networks and Adam moments,
float64 estimators / PPO loss math / SAC targets / normalizer statistics, so
that it reproduces the reference to ~1 ulp (checked against golden vectors
produced by the reference itself, tests/test_oracle_pinned.py).

Networks are represented as a small ``Net`` record: ``layers`` is a list of
``[W (out,in), b (out,)]`` pairs plus ``log_std``; the flat order
(W0, b0, W1, b1, ..., log_std) matches ``ModelParams.flat``
(R:tensornet/mlp.py:53-57) and ``Grads.flat`` (:93-96).
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field

import numpy as np

LOG_2PI = math.log(2.0 * math.pi)
SQUASH_EPS = 1e-6
NORM_CLIP = 10.0
NORM_EPS = 1e-8


class Diverged(RuntimeError):
    """Oracle analogue of the reference ``DivergenceError``."""


# ---------------------------------------------------------------- rng streams
def philox_stream(seed: int, label: str) -> np.random.Generator:
    """Named Philox stream keyed by blake2b("{seed}/{label}") (R:envcore/rng.py:17-26)."""
    key = int.from_bytes(
        hashlib.blake2b(f"{seed}/{label}".encode(), digest_size=16).digest(), "little"
    )
    return np.random.Generator(np.random.Philox(key=key))


# ------------------------------------------------------------------- networks
@dataclass
class Net:
    dims: tuple            # (in, h1, ..., out)
    layers: list           # [[W, b], ...]
    log_std: np.ndarray
    # builder extension (not in the reference): [[g, beta], ...] per hidden
    # layer when the net has LayerNorm; flat order W, b, g, beta per layer
    ln: list = field(default_factory=list)

    def pairs(self) -> list:
        """Parameter pairs in flat order: [W0,b0], [g0,beta0]?, [W1,b1], ..."""
        out = []
        for i, pair in enumerate(self.layers):
            out.append(pair)
            if i < len(self.ln):
                out.append(self.ln[i])
        return out

    def arrays(self) -> list:
        return [a for pair in self.pairs() for a in pair] + [self.log_std]

    def flat(self) -> np.ndarray:
        return np.concatenate([a.ravel() for a in self.arrays()])

    def load_flat(self, vec: np.ndarray) -> "Net":
        out = self.clone()
        pos = 0
        for pair in out.pairs():
            for j in range(2):
                n = pair[j].size
                pair[j] = vec[pos:pos + n].reshape(pair[j].shape).astype(pair[j].dtype)
                pos += n
        out.log_std = vec[pos:pos + out.log_std.size].astype(out.log_std.dtype)
        return out

    def clone(self) -> "Net":
        return Net(self.dims, [[w.copy(), b.copy()] for w, b in self.layers],
                   self.log_std.copy(), [[g.copy(), b.copy()] for g, b in self.ln])

    def zeros(self) -> "Net":
        return Net(self.dims, [[np.zeros_like(w), np.zeros_like(b)] for w, b in self.layers],
                   np.zeros_like(self.log_std),
                   [[np.zeros_like(g), np.zeros_like(b)] for g, b in self.ln])


class _Acts(list):
    """Hidden activations; .ln holds the LayerNorm caches of an LN net."""

    ln: list


def net_init(dims, seed: int, noise_std: float = 1.0, dtype=np.float32,
             layer_norm: bool = False) -> Net:
    """U(+-sqrt(1/fan_in)) weights drawn layer by layer from default_rng(seed), zero
    biases, log_std = ln(noise_std) (R:tensornet/mlp.py:116-131).  layer_norm
    (extension) adds gain 1 / shift 0 per hidden layer, drawing nothing."""
    gen = np.random.default_rng(seed)
    layers = []
    for fan_in, fan_out in zip(dims[:-1], dims[1:]):
        lim = np.sqrt(1.0 / fan_in)
        layers.append([gen.uniform(-lim, lim, (fan_out, fan_in)).astype(dtype),
                       np.zeros(fan_out, dtype=dtype)])
    ln = [[np.ones(d, dtype), np.zeros(d, dtype)] for d in dims[1:-1]] if layer_norm else []
    return Net(tuple(dims), layers, np.full(dims[-1], np.log(noise_std), dtype=dtype), ln)


def elu(z):
    """expm1(clip(z,-60,0)) + max(z,0) (R:tensornet/mlp.py:134-138)."""
    return np.expm1(np.clip(z, -60.0, 0)) + np.maximum(z, 0)


def elu_grad_from_act(h):
    """min(h,0)+1 (R:tensornet/mlp.py:141-143)."""
    return np.minimum(h, 0) + 1.0


def mlp_forward(net: Net, x):
    """z = h W^T + b; ELU on hidden layers (R:tensornet/mlp.py:153-172).
    Returns (out, acts) with acts = hidden activations (the cache backward uses)."""
    x = np.asarray(x)
    if x.ndim != 2 or x.shape[1] != net.dims[0]:
        raise ValueError("input width mismatch")
    acts = _Acts()
    acts.ln = []
    h = x
    last = len(net.layers) - 1
    for i, (w, b) in enumerate(net.layers):
        z = h @ w.T + b
        if i < last:
            if net.ln:  # extension: z -> LN(z) g + beta before the ELU
                n, cache = ln_forward(z, net.ln[i][0], net.ln[i][1])
                acts.ln.append(cache)
                z = n.astype(z.dtype)
            h = elu(z)
            acts.append(h)
        else:
            h = z
    return h, acts


def mlp_backward(net: Net, x, acts, dout):
    """Reverse mode through the cached forward (R:tensornet/mlp.py:175-198).
    dout is cast to the parameter dtype first (:186-187); dX of layer 0 is
    produced as well (:195)."""
    g = net.zeros()
    dh = np.asarray(dout, dtype=net.layers[-1][0].dtype)
    for i in range(len(net.layers) - 1, -1, -1):
        w = net.layers[i][0]
        inp = x if i == 0 else acts[i - 1]
        g.layers[i][0] += dh.T @ inp
        g.layers[i][1] += dh.sum(axis=0)
        dh = dh @ w
        if i > 0:
            dh = dh * elu_grad_from_act(acts[i - 1])
            if net.ln:
                dz, dg, db = ln_backward(dh, net.ln[i - 1][0], acts.ln[i - 1])
                g.ln[i - 1][0] += dg.astype(g.ln[i - 1][0].dtype)
                g.ln[i - 1][1] += db.astype(g.ln[i - 1][1].dtype)
                dh = dz.astype(dh.dtype)
    return dh, g


def value_forward(net: Net, x):
    out, acts = mlp_forward(net, x)
    return out[:, 0], acts


# ------------------------------------------------------------- distributions
def gauss_logp(mean, log_std, action):
    """sum_j(-log_std - 0.5 ln 2pi - 0.5 z^2) (R:tensornet/distributions.py:11-18)."""
    z = (np.asarray(action) - np.asarray(mean)) / np.exp(log_std)
    return (-log_std - 0.5 * LOG_2PI - 0.5 * z * z).sum(axis=-1)


def gauss_entropy(log_std) -> float:
    """sum(log_std + 0.5 (ln 2pi + 1)) (R:tensornet/distributions.py:21-26)."""
    return float(np.sum(log_std + 0.5 * (LOG_2PI + 1.0)))


def squash_logp(mean, log_std, u, a):
    """Gaussian logp of u minus sum log1p(-a^2 + 1e-6) (R:tensornet/distributions.py:66-70)."""
    return gauss_logp(mean, log_std, u) - np.log1p(-(a * a) + SQUASH_EPS).sum(axis=-1)


def squash_sample(mean, log_std, eps):
    """a = tanh(mean + std*eps), eps cast to mean dtype (R:tensornet/distributions.py:73-84)."""
    mean = np.asarray(mean)
    u = mean + np.exp(log_std) * np.asarray(eps, dtype=mean.dtype)
    a = np.tanh(u)
    return a, u, squash_logp(mean, log_std, u, a)


# ---------------------------------------------------------------- estimators
def _bootstrap_next(values, bootstrap, truncated, truncation_values):
    """V(s_{t+1}) with the truncation override (R:algos/estimators.py:15-26)."""
    nxt = np.concatenate([values[1:], bootstrap[None, :]], axis=0)
    if truncated is not None and truncation_values is not None:
        nxt = np.where(truncated, truncation_values, nxt)
    return nxt


def gae(rewards, values, terminated, truncated, bootstrap, gamma, lam,
        truncation_values=None):
    """f64 reverse GAE scan (R:algos/estimators.py:29-63)."""
    r = np.asarray(rewards, np.float64)
    v = np.asarray(values, np.float64)
    term = np.asarray(terminated, bool)
    trunc = np.asarray(truncated, bool)
    boot = np.asarray(bootstrap, np.float64)
    if not (r.shape == v.shape == term.shape == trunc.shape):
        raise ValueError("rewards/values/terminated/truncated must share (T, B)")
    nxt = _bootstrap_next(v, boot, trunc, truncation_values)
    delta = r + gamma * (~term) * nxt - v
    keep = ~(term | trunc)
    adv = np.zeros_like(r)
    run = np.zeros(r.shape[1])
    for t in reversed(range(r.shape[0])):
        run = delta[t] + gamma * lam * keep[t] * run
        adv[t] = run
    return adv, adv + v


def vtrace(behavior_logp, target_logp, rewards, values, terminated, bootstrap,
           gamma, rho_bar, c_bar, truncated=None, truncation_values=None):
    """f64 V-trace reverse scan (R:algos/estimators.py:66-122)."""
    bl = np.asarray(behavior_logp, np.float64)
    tl = np.asarray(target_logp, np.float64)
    r = np.asarray(rewards, np.float64)
    v = np.asarray(values, np.float64)
    term = np.asarray(terminated, bool)
    boot = np.asarray(bootstrap, np.float64)
    if not (r.shape == v.shape == term.shape == bl.shape == tl.shape):
        raise ValueError("vtrace inputs must share (T, B)")
    trunc = np.zeros_like(term) if truncated is None else np.asarray(truncated, bool)
    done = term | trunc
    ratio = np.exp(tl - bl)
    rho = np.minimum(rho_bar, ratio)
    c = np.minimum(c_bar, ratio)
    nxt = _bootstrap_next(v, boot, trunc, truncation_values)
    delta = rho * (r + gamma * (~term) * nxt - v)
    vs = np.zeros_like(r)
    carry = np.zeros(r.shape[1])
    for t in reversed(range(r.shape[0])):
        vs[t] = v[t] + delta[t] + gamma * (~done[t]) * c[t] * carry
        carry = vs[t] - v[t]
    vs_next = np.concatenate([vs[1:], boot[None, :]], axis=0)
    pg = rho * (r + gamma * (~term) * np.where(done, nxt, vs_next) - v)
    return vs, pg


# ------------------------------------------------------------------ optimizer
@dataclass
class Opt:
    m: Net
    v: Net
    t: int = 0
    lr: float = 1e-3
    b1: float = 0.9
    b2: float = 0.999
    eps: float = 1e-8

    @staticmethod
    def for_net(net: Net, lr: float) -> "Opt":
        return Opt(net.zeros(), net.zeros(), 0, lr)


def grad_norm(g: Net) -> float:
    """sqrt(sum over arrays of float(sum(a*a))) (R:tensornet/mlp.py:104-107)."""
    return float(np.sqrt(sum(float(np.sum(a * a)) for a in g.arrays())))


def clip_norm(grads: list, max_norm: float) -> float:
    """Joint global-norm clip, in place; returns the pre-clip norm
    (R:tensornet/adam.py:30-40)."""
    total = float(np.sqrt(sum(grad_norm(g) ** 2 for g in grads)))
    if max_norm > 0 and total > max_norm:
        f = max_norm / (total + 1e-12)
        for g in grads:
            for pair in g.pairs():
                pair[0] *= f
                pair[1] *= f
            g.log_std *= f
    return total


def adam(net: Net, g: Net, opt: Opt, max_norm: float = 0.0) -> None:
    """Bias-corrected Adam, order W,b per layer then log_std (R:tensornet/adam.py:43-80)."""
    if not np.all(np.isfinite(g.flat())):
        raise Diverged("non-finite gradients in adam_step")
    if max_norm > 0:
        clip_norm([g], max_norm)
    opt.t += 1
    bc1 = 1.0 - opt.b1 ** opt.t
    bc2 = 1.0 - opt.b2 ** opt.t

    def one(p, gr, m, v):
        m *= opt.b1
        m += (1 - opt.b1) * gr
        v *= opt.b2
        v += (1 - opt.b2) * gr * gr
        p -= (opt.lr * (m / bc1) / (np.sqrt(v / bc2) + opt.eps)).astype(p.dtype)

    for p, gp, mp, vp in zip(net.pairs(), g.pairs(), opt.m.pairs(), opt.v.pairs()):
        for j in range(2):
            one(p[j], gp[j], mp[j], vp[j])
    one(net.log_std, g.log_std, opt.m.log_std, opt.v.log_std)


def scalar_adam(state: dict, x: float, g: float) -> float:
    """ScalarAdam.step in python floats (R:algos/sac.py:35-53)."""
    if not np.isfinite(g):
        raise Diverged("non-finite gradient in ScalarAdam")
    state["t"] += 1
    b1, b2 = 0.9, 0.999
    state["m"] = b1 * state["m"] + (1 - b1) * g
    state["v"] = b2 * state["v"] + (1 - b2) * g * g
    m_hat = state["m"] / (1 - b1 ** state["t"])
    v_hat = state["v"] / (1 - b2 ** state["t"])
    return x - state["lr"] * m_hat / (np.sqrt(v_hat) + 1e-8)


# ------------------------------------------------------------------------ PPO
@dataclass
class PpoCfg:
    clip_param: float = 0.2
    entropy_coef: float = 0.01
    value_loss_coef: float = 1.0
    use_clipped_value_loss: bool = True
    epochs: int = 5
    minibatches: int = 4
    lr: float = 1e-3
    gamma: float = 0.99
    lam: float = 0.95
    max_grad_norm: float = 1.0
    vtrace_clip_rho: float = 1.0
    vtrace_clip_c: float = 1.0


def ppo_loss_grads(actor: Net, critic: Net, obs, cobs, act, blogp, adv, ret, oldv,
                   cfg: PpoCfg):
    """Clipped surrogate + clipped value loss + entropy with exact grads
    (R:algos/ppo.py:70-129)."""
    n = obs.shape[0]
    eps = cfg.clip_param
    mean, a_acts = mlp_forward(actor, obs)
    logp = gauss_logp(mean, actor.log_std, act)
    ratio = np.exp(logp - blogp)
    s1 = ratio * adv
    s2 = np.clip(ratio, 1 - eps, 1 + eps) * adv
    policy_loss = -float(np.mean(np.minimum(s1, s2)))
    dlogp = np.where(s1 <= s2, -adv * ratio / n, 0.0)
    std = np.exp(actor.log_std)
    z = (act - mean) / std
    dmean = dlogp[:, None] * z / std
    dls = (dlogp[:, None] * (z * z - 1.0)).sum(axis=0) - cfg.entropy_coef
    entropy = gauss_entropy(actor.log_std)
    _, ga = mlp_backward(actor, obs, a_acts, dmean)
    ga.log_std += dls.astype(ga.log_std.dtype)

    v, c_acts = value_forward(critic, cobs)
    if cfg.use_clipped_value_loss:
        vc = oldv + np.clip(v - oldv, -eps, eps)
        lu = (v - ret) ** 2
        lc = (vc - ret) ** 2
        value_loss = float(np.mean(np.maximum(lu, lc)))
        dv = np.where(lu >= lc, 2.0 * (v - ret) / n, 0.0)
    else:
        value_loss = float(np.mean((v - ret) ** 2))
        dv = 2.0 * (v - ret) / n
    dv = dv * cfg.value_loss_coef
    _, gc = mlp_backward(critic, cobs, c_acts, dv[:, None])
    total = policy_loss + cfg.value_loss_coef * value_loss - cfg.entropy_coef * entropy
    terms = dict(policy_loss=policy_loss, value_loss=value_loss, entropy=entropy,
                 total=total, kl=float(np.mean(blogp - logp)))
    return terms, ga, gc


def normalize_adv(adv):
    """(A - mean)/(std + 1e-8), population std (R:algos/ppo.py:132-133)."""
    return (adv - adv.mean()) / (adv.std() + 1e-8)


def ppo_epochs(actor, critic, opt_a: Opt, opt_c: Opt, cfg: PpoCfg, rng, obs, cobs, act,
               blogp, adv, ret, oldv, perms=None):
    """Epoch x minibatch loop (R:algos/ppo.py:136-199).  ``perms`` may carry
    precomputed per-epoch permutations (same values rng.permutation gives)."""
    n = obs.shape[0]
    if n % cfg.minibatches:
        raise ValueError(f"minibatches {cfg.minibatches} must divide batch size {n}")
    mb = n // cfg.minibatches
    adv = normalize_adv(adv)
    sums = dict(policy_loss=0.0, value_loss=0.0, entropy=0.0)
    kls = []
    gnorm = 0.0
    for e in range(cfg.epochs):
        perm = rng.permutation(n) if perms is None else perms[e]
        kl_last = 0.0
        for k in range(cfg.minibatches):
            idx = perm[k * mb:(k + 1) * mb]
            terms, ga, gc = ppo_loss_grads(actor, critic, obs[idx], cobs[idx], act[idx],
                                           blogp[idx], adv[idx], ret[idx], oldv[idx], cfg)
            if not np.isfinite(terms["total"]):
                raise Diverged(f"non-finite PPO loss: {terms}")
            gnorm = clip_norm([ga, gc], cfg.max_grad_norm)
            adam(actor, ga, opt_a)
            adam(critic, gc, opt_c)
            for key in sums:
                sums[key] += terms[key]
            kl_last = terms["kl"]
        kls.append(kl_last)
    nb = cfg.epochs * cfg.minibatches
    return dict(policy_loss=sums["policy_loss"] / nb, value_loss=sums["value_loss"] / nb,
                entropy=sums["entropy"] / nb, kl=float(np.mean(kls)), lr=opt_a.lr,
                grad_norm=gnorm)


def _flat_rows(a):
    return a.reshape(-1, *a.shape[2:])


def ppo_update(seg: dict, actor, critic, opt_a, opt_c, cfg: PpoCfg, rng, perms=None):
    """(R:algos/ppo.py:202-229): segment must carry advantages/returns."""
    if seg.get("advantages") is None or seg.get("returns") is None:
        raise ValueError("segment advantages/returns not computed")
    return ppo_epochs(actor, critic, opt_a, opt_c, cfg, rng, _flat_rows(seg["obs"]),
                      _flat_rows(seg["critic_obs"]), _flat_rows(seg["actions"]),
                      seg["behavior_log_prob"].reshape(-1), seg["advantages"].reshape(-1),
                      seg["returns"].reshape(-1), seg["values"].reshape(-1), perms)


def appo_update(seg: dict, actor, critic, opt_a, opt_c, cfg: PpoCfg, rng,
                learner_version=0, perms=None):
    """Recompute target logp / values, V-trace, then the PPO loop on
    (pg_adv, vs, values_now) (R:algos/appo.py:21-70)."""
    t, b = seg["rewards"].shape
    obs, cobs, act = (_flat_rows(seg[k]) for k in ("obs", "critic_obs", "actions"))
    mean, _ = mlp_forward(actor, obs)
    tlogp = gauss_logp(mean, actor.log_std, act).reshape(t, b)
    v_now, _ = value_forward(critic, cobs)
    v_now = v_now.reshape(t, b).astype(np.float64)
    vs, pg = vtrace(seg["behavior_log_prob"], tlogp, seg["rewards"], v_now,
                    seg["terminated"], seg["bootstrap_value"], cfg.gamma,
                    cfg.vtrace_clip_rho, cfg.vtrace_clip_c, truncated=seg["truncated"],
                    truncation_values=seg.get("truncation_values"))
    st = ppo_epochs(actor, critic, opt_a, opt_c, cfg, rng, obs, cobs, act,
                    seg["behavior_log_prob"].reshape(-1), pg.reshape(-1), vs.reshape(-1),
                    v_now.reshape(-1), perms)
    st["staleness"] = learner_version - seg.get("behavior_version", 0)
    return st


def adaptive_lr(lr, kl, update_index, desired_kl=0.01, beta=0.9, grow=1.1, decay=1.2,
                interval=5, schedule="adaptive"):
    """Dead-band adaptive LR every ``interval`` updates (R:algos/ppo.py:232-250)."""
    if schedule != "adaptive" or update_index % interval:
        return lr
    if kl > desired_kl / beta:
        lr = lr / decay
    elif kl < desired_kl * beta:
        lr = lr * grow
    return float(np.clip(lr, 1e-6, 1e-2))


# ------------------------------------------------------------------------ SAC
@dataclass
class SacCfg:
    gamma: float = 0.97
    tau: float = 0.125
    actor_lr: float = 3e-4
    critic_lr: float = 3e-4
    alpha_lr: float = 3e-4
    alpha_init: float = 0.01
    target_entropy_ratio: float = 0.0
    policy_frequency: int = 4
    max_grad_norm: float = 0.0


@dataclass
class SacSt:
    actor: Net
    q1: Net
    q2: Net
    q1t: Net
    q2t: Net
    log_alpha: float
    opt_actor: Opt
    opt_q1: Opt
    opt_q2: Opt
    opt_alpha: dict
    act_dim: int
    count: int = 0

    @staticmethod
    def create(actor, q1, q2, cfg: SacCfg) -> "SacSt":
        return SacSt(actor, q1, q2, q1.clone(), q2.clone(), float(np.log(cfg.alpha_init)),
                     Opt.for_net(actor, cfg.actor_lr), Opt.for_net(q1, cfg.critic_lr),
                     Opt.for_net(q2, cfg.critic_lr),
                     dict(lr=cfg.alpha_lr, m=0.0, v=0.0, t=0), actor.dims[-1])


def polyak(target: Net, online: Net, tau: float) -> None:
    """target <- (1-tau) target + tau online, in place (R:algos/sac.py:100-108)."""
    for tp, op in zip(target.pairs(), online.pairs()):
        for j in range(2):
            tp[j] *= 1.0 - tau
            tp[j] += tau * op[j]
    target.log_std *= 1.0 - tau
    target.log_std += tau * online.log_std


def sac_target(st: SacSt, batch: dict, gamma: float, rng) -> np.ndarray:
    """y = r + gamma^n_used (1-term)(min(Q1t,Q2t) - alpha logpi) (R:algos/sac.py:111-125)."""
    nobs = batch["next_obs"]
    mean, _ = mlp_forward(st.actor, nobs)
    eps = rng.standard_normal(mean.shape)
    a, _, logp = squash_sample(mean, st.actor.log_std, eps)
    qin = np.concatenate([nobs, a], axis=-1)
    q1, _ = value_forward(st.q1t, qin)
    q2, _ = value_forward(st.q2t, qin)
    soft = np.minimum(q1, q2) - np.exp(st.log_alpha) * logp
    keep = 1.0 - batch["terminated"].astype(np.float64)
    return batch["reward"] + gamma ** batch["n_used"] * keep * soft


def critic_loss_grads(q: Net, qin, y):
    """MSE vs fixed target (R:algos/sac.py:128-136)."""
    n = qin.shape[0]
    pred, acts = value_forward(q, qin)
    err = pred - y
    _, g = mlp_backward(q, qin, acts, (2.0 * err / n)[:, None])
    return float(np.mean(err * err)), g, pred


def actor_loss_grads(st: SacSt, obs, eps):
    """Reparameterized actor loss with exact grads (R:algos/sac.py:181-221)."""
    n = obs.shape[0]
    alpha = float(np.exp(st.log_alpha))
    mean, a_acts = mlp_forward(st.actor, obs)
    a, _, logp = squash_sample(mean, st.actor.log_std, eps)
    qin = np.concatenate([obs, a], axis=-1)
    q1, c1 = value_forward(st.q1, qin)
    q2, c2 = value_forward(st.q2, qin)
    loss = float(np.mean(alpha * logp - np.minimum(q1, q2)))
    pick = (q1 <= q2).astype(np.float64)
    d1, _ = mlp_backward(st.q1, qin, c1, pick[:, None])
    d2, _ = mlp_backward(st.q2, qin, c2, (1.0 - pick)[:, None])
    dq_da = (d1 + d2)[:, obs.shape[1]:]
    std = np.exp(st.actor.log_std)
    oma = 1.0 - a * a
    dlogp_du = 2.0 * a * oma / (oma + SQUASH_EPS)
    du_dls = std * eps
    dmean = (alpha * dlogp_du - dq_da * oma) / n
    dls = ((alpha * (-1.0 + dlogp_du * du_dls) - dq_da * oma * du_dls) / n).sum(axis=0)
    _, g = mlp_backward(st.actor, obs, a_acts, dmean)
    g.log_std += dls.astype(g.log_std.dtype)
    return loss, g, logp


def alpha_loss_grad(log_alpha, logp, target_entropy):
    """(-log_alpha * mean(logp + H), -mean(logp + H)) (R:algos/sac.py:224-229)."""
    ex = float(np.mean(logp + target_entropy))
    return -log_alpha * ex, -ex


def sac_update(batch: dict, st: SacSt, cfg: SacCfg, rng) -> dict:
    """Target -> q1 Adam -> q2 Adam -> [actor + alpha] -> Polyak (R:algos/sac.py:139-178,
    232-249)."""
    n = batch["obs"].shape[0]
    if n < 2:
        raise ValueError("sac_update needs a batch of at least 2 rows")
    y = sac_target(st, batch, cfg.gamma, rng)
    qin = np.concatenate([batch["obs"], batch["action"]], axis=-1)
    closs = 0.0
    for q, o in ((st.q1, st.opt_q1), (st.q2, st.opt_q2)):
        l, g, _ = critic_loss_grads(q, qin, y)
        closs += l
        adam(q, g, o, cfg.max_grad_norm)
    if not np.isfinite(closs):
        raise Diverged(f"non-finite SAC critic loss {closs}")
    st.count += 1
    out = dict(critic_loss=closs, alpha=float(np.exp(st.log_alpha)))
    if st.count % cfg.policy_frequency == 0:
        eps = rng.standard_normal((n, st.act_dim))
        aloss, ga, logp = actor_loss_grads(st, batch["obs"], eps)
        if not np.isfinite(aloss):
            raise Diverged(f"non-finite SAC actor loss {aloss}")
        adam(st.actor, ga, st.opt_actor, cfg.max_grad_norm)
        te = -cfg.target_entropy_ratio * st.act_dim
        al, dla = alpha_loss_grad(st.log_alpha, logp, te)
        st.log_alpha = scalar_adam(st.opt_alpha, st.log_alpha, dla)
        out.update(actor_loss=aloss, alpha_loss=al, alpha=float(np.exp(st.log_alpha)))
    polyak(st.q1t, st.q1, cfg.tau)
    polyak(st.q2t, st.q2, cfg.tau)
    return out


# ----------------------------------------------------------------- normalizer
@dataclass
class NormStats:
    dim: int
    count: float = 0.0
    mean: np.ndarray = None
    var: np.ndarray = None
    frozen: bool = False

    def __post_init__(self):
        if self.mean is None:
            self.mean = np.zeros(self.dim)
        if self.var is None:
            self.var = np.zeros(self.dim)


def norm_update(ns: NormStats, batch) -> None:
    """Chan merge of batch mean / population var into f64 running stats
    (R:tensornet/normalizer.py:27-45)."""
    if ns.frozen:
        return
    x = np.asarray(batch, np.float64)
    n = x.shape[0]
    if n == 0:
        return
    bm, bv = x.mean(axis=0), x.var(axis=0)
    tot = ns.count + n
    d = bm - ns.mean
    new_mean = ns.mean + d * (n / tot)
    new_var = (ns.var * ns.count + bv * n + d * d * (ns.count * n / tot)) / tot
    ns.mean, ns.var, ns.count = new_mean, new_var, tot


def norm_apply(ns: NormStats, batch) -> np.ndarray:
    """clip((x-mu)/sqrt(var+1e-8), +-10) -> f32 (R:tensornet/normalizer.py:47-49)."""
    out = (np.asarray(batch) - ns.mean) / np.sqrt(ns.var + NORM_EPS)
    return np.clip(out, -NORM_CLIP, NORM_CLIP).astype(np.float32)


# -------------------------------------------------------------- replay ring
def codec_width(obs_dim, act_dim):
    """obs | action | reward | next_obs | terminated | n_used (R:replaypath/storage.py:17-46)."""
    return 2 * obs_dim + act_dim + 3


def codec_encode(obs_dim, act_dim, obs, action, reward, next_obs, terminated, n_used):
    d, a = obs_dim, act_dim
    rows = np.empty((len(obs), codec_width(d, a)), np.float32)
    rows[:, :d] = obs
    rows[:, d:d + a] = action
    rows[:, d + a] = reward
    rows[:, d + a + 1:2 * d + a + 1] = next_obs
    rows[:, 2 * d + a + 1] = np.asarray(terminated, np.float32)
    rows[:, 2 * d + a + 2] = np.asarray(n_used, np.float32)
    return rows


def codec_decode(obs_dim, act_dim, rows):
    d, a = obs_dim, act_dim
    return dict(obs=rows[:, :d], action=rows[:, d:d + a],
                reward=rows[:, d + a].astype(np.float64),
                next_obs=rows[:, d + a + 1:2 * d + a + 1],
                terminated=rows[:, 2 * d + a + 1] > 0.5,
                n_used=rows[:, 2 * d + a + 2].astype(np.int64))


class Ring:
    """Absolute-index row ring (R:replaypath/storage.py:49-133)."""

    def __init__(self, cap, width):
        if cap < 1:
            raise ValueError("capacity must be >= 1")
        self.cap, self.width, self.head = cap, width, 0
        self.data = np.zeros((cap, width), np.float32)

    def window(self):
        return max(0, self.head - self.cap), self.head

    def insert(self, rows):
        rows = np.asarray(rows, np.float32)
        if rows.ndim != 2 or rows.shape[1] != self.width:
            raise ValueError("row width incompatible with layout width")
        n = len(rows)
        ids = np.arange(self.head, self.head + n)
        if n >= self.cap:        # only the tail survives, at its own slots (:87-92)
            ids, rows = ids[-self.cap:], rows[-self.cap:]
        self.data[ids % self.cap] = rows
        self.head += n

    def read(self, idx):
        idx = np.asarray(idx, np.int64)
        lo, hi = self.window()
        if len(idx) and (idx.min() < lo or idx.max() >= hi):
            raise IndexError(f"row indices outside valid window [{lo}, {hi})")
        return self.data[idx % self.cap].copy()

    def sample_indices(self, batch, rng):
        lo, hi = self.window()
        if hi == lo:
            raise ValueError("replay empty")
        return rng.integers(lo, hi, size=batch)


# ------------------------------------------------- LayerNorm (builder oracle)
def ln_forward(x, g, b, eps=1e-5):
    """Row LayerNorm in f64.  NOT in the reference (R:tensornet/mlp.py:27-28 is
    ELU-only): parity here is pinned by finite differences only."""
    x = np.asarray(x, np.float64)
    mu = x.mean(axis=1, keepdims=True)
    var = x.var(axis=1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + eps)
    xh = (x - mu) * rstd
    return xh * g + b, (xh, rstd)


def ln_backward(dy, g, cache):
    xh, rstd = cache
    dy = np.asarray(dy, np.float64)
    dg = (dy * xh).sum(axis=0)
    db = dy.sum(axis=0)
    dxh = dy * g
    dx = rstd * (dxh - dxh.mean(axis=1, keepdims=True)
                 - xh * (dxh * xh).mean(axis=1, keepdims=True))
    return dx, dg, db
