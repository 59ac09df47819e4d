"""Generate golden input/output vectors by running the UNMODIFIED reference.

Run in the build container (where /root/reference exists):

    OPENBLAS_NUM_THREADS=1 python tests/golden/gen_golden.py

It imports ``unilite`` read-only from /root/reference/pkg/src and writes small
``.npz`` fixtures next to this script.  The fixtures travel with the repo; the
GPU box never needs /root/reference.  Each case stores the inputs it fed the
reference and the reference's outputs; ``tests/test_oracle_pinned.py`` pins the
numpy oracle against them and the ``-m gpu`` tests pin the CUDA path.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

import numpy as np  # noqa: E402

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

from unilite.algos import (  # noqa: E402
    AcOpt, AcParams, AppoConfig, PpoConfig, RolloutSegment, SacConfig, SacState,
    appo_update, critic_target, gae, ppo_loss_and_grads, ppo_update, sac_update, vtrace,
)
from unilite.envcore.rng import stream  # noqa: E402
from unilite.replaypath import ReplayStorage, RowCodec  # noqa: E402
from unilite.tensornet import (  # noqa: E402
    Arch, Normalizer, OptState, adam_step, backward, clip_global_norm, forward,
    gaussian_log_prob, init_params, value_forward,
)


def _scan_instance(rng, t, b, p_done=0.15):
    r = rng.normal(size=(t, b))
    v = rng.normal(size=(t, b))
    term = rng.random((t, b)) < p_done / 2
    trunc = (rng.random((t, b)) < p_done / 2) & ~term
    boot = rng.normal(size=b)
    tv = rng.normal(size=(t, b)) * trunc
    return r, v, term, trunc, boot, tv


def gen_scans():
    rng = np.random.default_rng(100)
    out = {}
    shapes = [(1, 1), (1, 7), (5, 1), (8, 3), (24, 64), (17, 33), (64, 5)]
    for i, (t, b) in enumerate(shapes):
        r, v, term, trunc, boot, tv = _scan_instance(rng, t, b)
        gamma, lam = float(rng.uniform(0.5, 1.0)), float(rng.uniform(0.0, 1.0))
        use_tv = i % 2 == 0
        adv, ret = gae(r, v, term, trunc, boot, gamma, lam,
                       truncation_values=tv if use_tv else None)
        bl = rng.normal(size=(t, b))
        tl = bl + rng.normal(scale=0.5, size=(t, b))
        rho_bar, c_bar = float(rng.uniform(0.5, 2.0)), float(rng.uniform(0.5, 2.0))
        vs, pg = vtrace(bl, tl, r, v, term, boot, gamma, rho_bar, c_bar,
                        truncated=trunc if i % 3 else None,
                        truncation_values=tv if use_tv else None)
        out.update({
            f"c{i}_r": r, f"c{i}_v": v, f"c{i}_term": term, f"c{i}_trunc": trunc,
            f"c{i}_boot": boot, f"c{i}_tv": tv, f"c{i}_use_tv": use_tv,
            f"c{i}_vt_trunc": bool(i % 3), f"c{i}_gamma": gamma, f"c{i}_lam": lam,
            f"c{i}_bl": bl, f"c{i}_tl": tl, f"c{i}_rho": rho_bar, f"c{i}_c": c_bar,
            f"c{i}_adv": adv, f"c{i}_ret": ret, f"c{i}_vs": vs, f"c{i}_pg": pg,
        })
    out["n_cases"] = len(shapes)
    np.savez_compressed(OUT / "scans.npz", **out)


def gen_mlp():
    out = {}
    rng = np.random.default_rng(200)
    cases = [((5, (7, 6), 3), np.float32), ((4, (), 2), np.float64), ((9, (16, 8, 4), 1), np.float32)]
    for i, ((din, hid, dout), dt) in enumerate(cases):
        p = init_params(Arch(din, hid, dout), seed=10 + i, dtype=dt)
        x = rng.normal(size=(11, din)).astype(dt)
        y, cache = forward(p, x)
        g_out = rng.normal(size=y.shape)
        dx, grads = backward(p, cache, g_out)
        out.update({f"c{i}_dims": np.array([din, *hid, dout]), f"c{i}_f64": dt == np.float64,
                    f"c{i}_params": p.flat(), f"c{i}_x": x, f"c{i}_y": y, f"c{i}_dout": g_out,
                    f"c{i}_dx": dx, f"c{i}_grads": grads.flat()})
    out["n_cases"] = len(cases)
    np.savez_compressed(OUT / "mlp.npz", **out)


def gen_adam():
    rng = np.random.default_rng(300)
    p = init_params(Arch(6, (8,), 3), seed=3)
    opt = OptState.for_params(p, lr=1e-3)
    out = {"params0": p.flat()}
    for s in range(4):
        _, g = backward(p, forward(p, rng.normal(size=(5, 6)).astype(np.float32))[1],
                        rng.normal(size=(5, 3)) * (10.0 if s == 2 else 1.0))
        g.log_std += rng.normal(size=3).astype(np.float32)
        out[f"g{s}"] = g.flat()
        norm = clip_global_norm([g], 1.0) if s % 2 else 0.0
        out[f"norm{s}"] = norm
        out[f"gclipped{s}"] = g.flat()
        adam_step(p, g, opt, max_grad_norm=0.5 if s == 3 else 0.0)
        out[f"params{s + 1}"] = p.flat()
        out[f"m{s + 1}"] = opt.m.flat()
        out[f"v{s + 1}"] = opt.v.flat()
    np.savez_compressed(OUT / "adam.npz", **out)


def _synthetic_segment(t, b, od, cd, ad, hid, seed, perturb=0.0):
    """BASELINE.md synthetic-input recipe at a small size."""
    rng = np.random.default_rng(seed)
    actor = init_params(Arch(od, hid, ad), seed=0, init_noise_std=1.0)
    critic = init_params(Arch(cd, hid, 1), seed=1)
    obs = rng.normal(size=(t, b, od)).astype(np.float32)
    cobs = rng.normal(size=(t, b, cd)).astype(np.float32)
    act = rng.normal(size=(t, b, ad)).astype(np.float32)
    rew = 0.1 * rng.normal(size=(t, b))
    term = rng.random((t, b)) < 0.01 * 5
    trunc = (rng.random((t, b)) < 0.005 * 5) & ~term
    boot = rng.normal(size=b)
    tv = rng.normal(size=(t, b)) * trunc
    beh = actor.copy()
    if perturb:
        for w, bb in beh.layers:
            w += (perturb * rng.normal(size=w.shape)).astype(w.dtype)
    mean, _ = forward(beh, obs.reshape(-1, od))
    blogp = gaussian_log_prob(mean, beh.log_std, act.reshape(-1, ad)).reshape(t, b).astype(np.float64)
    vals, _ = value_forward(critic, cobs.reshape(-1, cd))
    vals = vals.reshape(t, b).astype(np.float64)
    seg = RolloutSegment(obs=obs, critic_obs=cobs, actions=act, behavior_log_prob=blogp,
                         rewards=rew, terminated=term, truncated=trunc, values=vals,
                         bootstrap_value=boot, truncation_values=tv, behavior_version=3)
    return seg, actor, critic


def _seg_dict(seg, prefix):
    keys = ["obs", "critic_obs", "actions", "behavior_log_prob", "rewards", "terminated",
            "truncated", "values", "bootstrap_value", "truncation_values"]
    return {f"{prefix}{k}": getattr(seg, k) for k in keys}


def gen_ppo():
    out = {}
    # (a) one PPO loss/grad step at a moderate size, f32 nets (the fp32 parity contract)
    seg, actor, critic = _synthetic_segment(6, 32, 10, 12, 4, (32, 16), seed=401)
    cfg = PpoConfig()
    adv, ret = gae(seg.rewards, seg.values, seg.terminated, seg.truncated,
                   seg.bootstrap_value, cfg.gamma, cfg.lam, truncation_values=seg.truncation_values)
    seg.advantages, seg.returns = adv, ret
    out.update(_seg_dict(seg, "s_"))
    out.update(s_adv=adv, s_ret=ret, s_actor=actor.flat(), s_critic=critic.flat())
    n = 6 * 32
    idx = np.arange(0, n, 3)
    flat = lambda a: a.reshape(-1, *a.shape[2:])
    advn = (adv.reshape(-1) - adv.mean()) / (adv.std() + 1e-8)
    terms, ga, gc = ppo_loss_and_grads(
        AcParams(actor, critic), flat(seg.obs)[idx], flat(seg.critic_obs)[idx],
        flat(seg.actions)[idx], seg.behavior_log_prob.reshape(-1)[idx], advn[idx],
        ret.reshape(-1)[idx], seg.values.reshape(-1)[idx], cfg)
    out.update(s_idx=idx, s_ga=ga.flat(), s_gc=gc.flat(),
               s_terms=np.array([terms[k] for k in ("policy_loss", "value_loss", "entropy", "total", "kl")]))
    # (b) a full ppo_update, reference stream(1,"update")
    seg, actor, critic = _synthetic_segment(8, 16, 6, 7, 3, (16, 16), seed=402)
    cfg = PpoConfig(epochs=2, minibatches=4)
    adv, ret = gae(seg.rewards, seg.values, seg.terminated, seg.truncated,
                   seg.bootstrap_value, cfg.gamma, cfg.lam, truncation_values=seg.truncation_values)
    seg.advantages, seg.returns = adv, ret
    out.update(_seg_dict(seg, "u_"))
    out.update(u_adv=adv, u_ret=ret, u_actor0=actor.flat(), u_critic0=critic.flat())
    params = AcParams(actor, critic)
    opt = AcOpt.for_params(params, cfg.lr)
    st = ppo_update(seg, params, opt, cfg, stream(1, "update"))
    out.update(u_actor1=params.actor.flat(), u_critic1=params.critic.flat(),
               u_ma=opt.actor.m.flat(), u_va=opt.actor.v.flat(),
               u_mc=opt.critic.m.flat(), u_vc=opt.critic.v.flat(),
               u_stats=np.array([st.policy_loss, st.value_loss, st.entropy, st.kl, st.lr, st.grad_norm]))
    # (c) appo_update with a perturbed behaviour policy
    seg, actor, critic = _synthetic_segment(8, 16, 6, 7, 3, (16, 16), seed=403, perturb=1e-2)
    cfg = AppoConfig(epochs=2, minibatches=2)
    out.update(_seg_dict(seg, "a_"))
    out.update(a_actor0=actor.flat(), a_critic0=critic.flat())
    params = AcParams(actor, critic)
    opt = AcOpt.for_params(params, cfg.lr)
    st = appo_update(seg, params, opt, cfg, stream(1, "update"), learner_version=5)
    out.update(a_actor1=params.actor.flat(), a_critic1=params.critic.flat(),
               a_stats=np.array([st.policy_loss, st.value_loss, st.entropy, st.kl, st.lr,
                                 st.grad_norm, st.staleness]))
    np.savez_compressed(OUT / "ppo.npz", **out)


def gen_sac():
    rng = np.random.default_rng(500)
    od, ad, hid = 5, 2, (16, 16)
    cfg = SacConfig(policy_frequency=2, batch_size=16)
    actor = init_params(Arch(od, hid, ad), seed=1, init_noise_std=1.0)
    q1 = init_params(Arch(od + ad, hid, 1), seed=2)
    q2 = init_params(Arch(od + ad, hid, 1), seed=3)
    state = SacState.create(actor, q1, q2, cfg)
    out = {"actor0": actor.flat(), "q10": q1.flat(), "q20": q2.flat()}
    lrng = stream(1, "learner")
    for s in range(4):
        batch = dict(obs=rng.normal(size=(16, od)).astype(np.float32),
                     action=np.tanh(rng.normal(size=(16, ad))).astype(np.float32),
                     reward=rng.normal(size=16),
                     next_obs=rng.normal(size=(16, od)).astype(np.float32),
                     terminated=rng.random(16) < 0.2,
                     n_used=rng.integers(1, 3, size=16).astype(np.int64))
        for k, v in batch.items():
            out[f"b{s}_{k}"] = v
        if s == 0:
            y = critic_target(state.params, batch, cfg.gamma, stream(9, "probe"))
            out["y0"] = y
        st = sac_update(batch, state, cfg, lrng)
        out[f"stats{s}"] = np.array([st.extra.get(k, np.nan) for k in
                                     ("critic_loss", "actor_loss", "alpha_loss", "alpha")])
        p = state.params
        out.update({f"actor{s + 1}": p.actor.flat(), f"q1{s + 1}": p.q1.flat(),
                    f"q2{s + 1}": p.q2.flat(), f"q1t{s + 1}": p.q1_targ.flat(),
                    f"q2t{s + 1}": p.q2_targ.flat(), f"log_alpha{s + 1}": p.log_alpha})
    np.savez_compressed(OUT / "sac.npz", **out)


def gen_normalizer_replay():
    rng = np.random.default_rng(600)
    out = {}
    norm = Normalizer(7)
    for s, n in enumerate([5, 1, 40, 0, 13]):
        x = (rng.normal(size=(n, 7)) * 3 + 1).astype(np.float32)
        norm.update(x)
        out[f"n_x{s}"] = x
        out[f"n_mean{s}"] = norm.mean.copy()
        out[f"n_var{s}"] = norm.var.copy()
        out[f"n_count{s}"] = norm.count
        out[f"n_apply{s}"] = norm.apply(x)
    codec = RowCodec(4, 2)
    storage = ReplayStorage(capacity=37, row_width=codec.width)
    head_rows = []
    for s, n in enumerate([5, 20, 11, 50, 3, 37]):
        rows = rng.normal(size=(n, codec.width)).astype(np.float32)
        storage.insert(rows)
        head_rows.append(rows)
        out[f"r_rows{s}"] = rows
    srng = stream(1, "replay")
    idx = storage.sample_indices(64, srng)
    out["r_idx"] = idx
    out["r_read"] = storage.read_rows(idx)
    out["r_window"] = np.array(storage.valid_range())
    out["r_snapshot"] = storage.snapshot_sample(16, stream(1, "replay2"))
    dec = codec.decode(out["r_read"])
    for k, v in dec.items():
        out[f"r_dec_{k}"] = v
    np.savez_compressed(OUT / "norm_replay.npz", **out)


def gen_perms():
    """The exact permutation stream ppo_update consumes (R:algos/ppo.py:162)."""
    rng = stream(1, "update")
    out = {f"perm{e}": rng.permutation(96) for e in range(3)}
    rng = stream(1, "replay")
    out["ints"] = rng.integers(100, 1000, size=50)
    np.savez_compressed(OUT / "perms.npz", **out)


if __name__ == "__main__":
    gen_scans()
    gen_mlp()
    gen_adam()
    gen_ppo()
    gen_sac()
    gen_normalizer_replay()
    gen_perms()
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)
