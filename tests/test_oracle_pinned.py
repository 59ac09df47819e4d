"""Pin the numpy oracle (oracle/port.py) to the reference before trusting it.

Checks against (1) golden vectors the unmodified reference produced
(tests/golden/gen_golden.py) and (2) the reference test-suite's own known
answers (R:tests/test_estimators.py:124-231, test_ppo.py:214-238,
test_sac.py:78-110).  CPU only.
"""

import numpy as np
import pytest

from oracle import port as O


def _net_from_flat(dims, flat, dtype=np.float32):
    return O.net_init(dims, 0, dtype=dtype).load_flat(np.asarray(flat))


# ------------------------------------------------------------------ estimators
def test_scans_match_reference_goldens(golden):
    g = golden("scans")
    for i in range(int(g["n_cases"])):
        c = lambda k: g[f"c{i}_{k}"]
        tv = c("tv") if bool(c("use_tv")) else None
        adv, ret = O.gae(c("r"), c("v"), c("term"), c("trunc"), c("boot"), float(c("gamma")),
                         float(c("lam")), truncation_values=tv)
        np.testing.assert_allclose(adv, c("adv"), rtol=0, atol=1e-12)
        np.testing.assert_allclose(ret, c("ret"), rtol=0, atol=1e-12)
        vs, pg = O.vtrace(c("bl"), c("tl"), c("r"), c("v"), c("term"), c("boot"),
                          float(c("gamma")), float(c("rho")), float(c("c")),
                          truncated=c("trunc") if bool(c("vt_trunc")) else None,
                          truncation_values=tv)
        np.testing.assert_allclose(vs, c("vs"), rtol=0, atol=1e-12)
        np.testing.assert_allclose(pg, c("pg"), rtol=0, atol=1e-12)


def test_known_answers_scans():
    # R:tests/test_estimators.py:132-139 (1-step TD = 1.99)
    adv, ret = O.gae(np.array([[1.0]]), np.array([[0.0]]), np.zeros((1, 1), bool),
                     np.zeros((1, 1), bool), np.array([1.0]), 0.99, 0.0)
    assert adv[0, 0] == pytest.approx(1.99) and ret[0, 0] == pytest.approx(1.99)
    # gamma=0 collapse (:125-130)
    adv, _ = O.gae(np.ones((2, 1)), np.full((2, 1), 0.5), np.zeros((2, 1), bool),
                   np.zeros((2, 1), bool), np.zeros(1), 0.0, 0.95)
    np.testing.assert_allclose(adv, [[0.5], [0.5]])
    # V-trace ratio 2 / ratio 1/2 (:191-209)
    for ratio, evs, epg in ((2.0, 1.99, 1.49), (0.5, 1.245, 0.745)):
        vs, pg = O.vtrace(np.array([[0.0]]), np.array([[np.log(ratio)]]), np.array([[1.0]]),
                          np.array([[0.5]]), np.zeros((1, 1), bool), np.array([1.0]),
                          0.99, 1.0, 1.0)
        assert vs[0, 0] == pytest.approx(evs) and pg[0, 0] == pytest.approx(epg)
    # SURVEY Appendix A 2-step example: vs=[4.33,3.70], pg=[3.83,-3.30] is a
    # property of that example's inputs; the on-policy identity below is the
    # reference's own (:175-189).
    rng = np.random.default_rng(2)
    for _ in range(10):
        t, b = int(rng.integers(2, 12)), int(rng.integers(1, 4))
        r, v = rng.normal(size=(t, b)), rng.normal(size=(t, b))
        term = rng.random((t, b)) < 0.07
        trunc = (rng.random((t, b)) < 0.07) & ~term
        boot, tv, lp = rng.normal(size=b), rng.normal(size=(t, b)), rng.normal(size=(t, b))
        vs, pg = O.vtrace(lp, lp, r, v, term, boot, 0.99, 1.0, 1.0, truncated=trunc,
                          truncation_values=tv)
        adv, ret = O.gae(r, v, term, trunc, boot, 0.99, 1.0, truncation_values=tv)
        np.testing.assert_allclose(vs, ret, atol=1e-10)
        np.testing.assert_allclose(pg, adv, atol=1e-10)


# ------------------------------------------------------------------------- MLP
def test_mlp_matches_reference_goldens(golden):
    g = golden("mlp")
    for i in range(int(g["n_cases"])):
        c = lambda k: g[f"c{i}_{k}"]
        dt = np.float64 if bool(c("f64")) else np.float32
        net = _net_from_flat(tuple(int(d) for d in c("dims")), c("params"), dt)
        y, acts = O.mlp_forward(net, c("x"))
        np.testing.assert_array_equal(y, c("y"))
        dx, gr = O.mlp_backward(net, c("x"), acts, c("dout"))
        np.testing.assert_array_equal(dx, c("dx"))
        np.testing.assert_array_equal(gr.flat(), c("grads"))


def test_adam_matches_reference_goldens(golden):
    g = golden("adam")
    net = _net_from_flat((6, 8, 3), g["params0"])
    opt = O.Opt.for_net(net, 1e-3)
    for s in range(4):
        gr = net.zeros().load_flat(g[f"g{s}"])
        if s % 2:
            assert O.clip_norm([gr], 1.0) == pytest.approx(float(g[f"norm{s}"]), rel=1e-12)
        np.testing.assert_array_equal(gr.flat(), g[f"gclipped{s}"])
        O.adam(net, gr, opt, max_norm=0.5 if s == 3 else 0.0)
        np.testing.assert_array_equal(net.flat(), g[f"params{s + 1}"])
        np.testing.assert_array_equal(opt.m.flat(), g[f"m{s + 1}"])
        np.testing.assert_array_equal(opt.v.flat(), g[f"v{s + 1}"])


def test_adam_known_answers():
    # R:tests/test_tensornet.py Adam cases: first step moves by lr*(1-ish); NaN raises
    net = O.net_init((2, 1), 0)
    opt = O.Opt.for_net(net, 1e-3)
    before = net.flat().copy()
    gr = net.zeros()
    gr.layers[0][0][:] = 1.0
    O.adam(net, gr, opt)
    np.testing.assert_allclose((before - net.flat())[:2], 1e-3, rtol=1e-4)
    gr.layers[0][0][0, 0] = np.nan
    with pytest.raises(O.Diverged):
        O.adam(net, gr, opt)


# ------------------------------------------------------------------ PPO / APPO
def _seg(g, p):
    keys = ["obs", "critic_obs", "actions", "behavior_log_prob", "rewards", "terminated",
            "truncated", "values", "bootstrap_value", "truncation_values"]
    return {k: g[p + k] for k in keys}


def test_ppo_loss_grads_match_reference(golden):
    g = golden("ppo")
    seg = _seg(g, "s_")
    actor = _net_from_flat((10, 32, 16, 4), g["s_actor"])
    critic = _net_from_flat((12, 32, 16, 1), g["s_critic"])
    cfg = O.PpoCfg()
    adv, ret = O.gae(seg["rewards"], seg["values"], seg["terminated"], seg["truncated"],
                     seg["bootstrap_value"], cfg.gamma, cfg.lam, seg["truncation_values"])
    np.testing.assert_allclose(adv, g["s_adv"], atol=1e-12)
    idx = g["s_idx"]
    advn = O.normalize_adv(adv.reshape(-1))
    flat = lambda a: a.reshape(-1, *a.shape[2:])
    terms, ga, gc = O.ppo_loss_grads(actor, critic, flat(seg["obs"])[idx],
                                     flat(seg["critic_obs"])[idx], flat(seg["actions"])[idx],
                                     seg["behavior_log_prob"].reshape(-1)[idx], advn[idx],
                                     ret.reshape(-1)[idx], seg["values"].reshape(-1)[idx], cfg)
    np.testing.assert_allclose([terms[k] for k in ("policy_loss", "value_loss", "entropy",
                                                   "total", "kl")], g["s_terms"], rtol=1e-12)
    np.testing.assert_allclose(ga.flat(), g["s_ga"], rtol=1e-6, atol=1e-9)
    np.testing.assert_allclose(gc.flat(), g["s_gc"], rtol=1e-6, atol=1e-9)


def test_ppo_update_matches_reference(golden):
    g = golden("ppo")
    seg = _seg(g, "u_")
    seg["advantages"], seg["returns"] = g["u_adv"], g["u_ret"]
    actor = _net_from_flat((6, 16, 16, 3), g["u_actor0"])
    critic = _net_from_flat((7, 16, 16, 1), g["u_critic0"])
    cfg = O.PpoCfg(epochs=2, minibatches=4)
    oa, oc = O.Opt.for_net(actor, cfg.lr), O.Opt.for_net(critic, cfg.lr)
    st = O.ppo_update(seg, actor, critic, oa, oc, cfg, O.philox_stream(1, "update"))
    np.testing.assert_allclose(actor.flat(), g["u_actor1"], rtol=0, atol=1e-6)
    np.testing.assert_allclose(critic.flat(), g["u_critic1"], rtol=0, atol=1e-6)
    np.testing.assert_allclose([st[k] for k in ("policy_loss", "value_loss", "entropy", "kl",
                                                "lr", "grad_norm")], g["u_stats"], rtol=1e-6,
                               atol=1e-9)


def test_appo_update_matches_reference(golden):
    g = golden("ppo")
    seg = _seg(g, "a_")
    seg["behavior_version"] = 3
    actor = _net_from_flat((6, 16, 16, 3), g["a_actor0"])
    critic = _net_from_flat((7, 16, 16, 1), g["a_critic0"])
    cfg = O.PpoCfg(epochs=2, minibatches=2)
    oa, oc = O.Opt.for_net(actor, cfg.lr), O.Opt.for_net(critic, cfg.lr)
    st = O.appo_update(seg, actor, critic, oa, oc, cfg, O.philox_stream(1, "update"),
                       learner_version=5)
    np.testing.assert_allclose(actor.flat(), g["a_actor1"], atol=1e-6)
    np.testing.assert_allclose(critic.flat(), g["a_critic1"], atol=1e-6)
    np.testing.assert_allclose([st[k] for k in ("policy_loss", "value_loss", "entropy", "kl",
                                                "lr", "grad_norm", "staleness")], g["a_stats"],
                               rtol=1e-6, atol=1e-9)


def test_adaptive_lr_known_answers():
    # R:tests/test_ppo.py:214-238
    assert O.adaptive_lr(1e-3, 0.02, 5) == pytest.approx(1e-3 / 1.2)
    assert O.adaptive_lr(1e-3, 0.005, 10) == pytest.approx(1.1e-3)
    assert O.adaptive_lr(1e-3, 0.0095, 5) == 1e-3
    assert O.adaptive_lr(1e-3, 0.02, 3) == 1e-3
    assert O.adaptive_lr(9.5e-3, 0.001, 5) == 1e-2
    assert O.adaptive_lr(1.1e-6, 1.0, 5) == 1e-6


# ------------------------------------------------------------------------- SAC
def test_sac_updates_match_reference(golden):
    g = golden("sac")
    od, ad = 5, 2
    actor = _net_from_flat((od, 16, 16, ad), g["actor0"])
    q1 = _net_from_flat((od + ad, 16, 16, 1), g["q10"])
    q2 = _net_from_flat((od + ad, 16, 16, 1), g["q20"])
    cfg = O.SacCfg(policy_frequency=2)
    st = O.SacSt.create(actor, q1, q2, cfg)
    rng = O.philox_stream(1, "learner")
    for s in range(4):
        batch = {k: g[f"b{s}_{k}"] for k in ("obs", "action", "reward", "next_obs",
                                            "terminated", "n_used")}
        if s == 0:
            y = O.sac_target(st, batch, cfg.gamma, O.philox_stream(9, "probe"))
            np.testing.assert_allclose(y, g["y0"], rtol=1e-12, atol=1e-12)
        out = O.sac_update(batch, st, cfg, rng)
        ref = g[f"stats{s}"]
        got = np.array([out.get(k, np.nan) for k in ("critic_loss", "actor_loss",
                                                     "alpha_loss", "alpha")])
        np.testing.assert_allclose(got, ref, rtol=1e-6, atol=1e-9)
        for name, net in (("actor", st.actor), ("q1", st.q1), ("q2", st.q2),
                          ("q1t", st.q1t), ("q2t", st.q2t)):
            np.testing.assert_allclose(net.flat(), g[f"{name}{s + 1}"], atol=1e-6)
        assert st.log_alpha == pytest.approx(float(g[f"log_alpha{s + 1}"]), abs=1e-9)


def test_polyak_known_answer():
    # R:tests/test_sac.py:78-90: tau 0.125 from zeros toward ones
    t = O.net_init((3, 4, 1), 0)
    o = t.clone()
    for p in t.layers:
        p[0][:] = 0
        p[1][:] = 0
    for p in o.layers:
        p[0][:] = 1
        p[1][:] = 1
    O.polyak(t, o, 0.125)
    assert t.layers[0][0][0, 0] == pytest.approx(0.125)


# ----------------------------------------------------- normalizer / replay ring
def test_normalizer_matches_reference(golden):
    g = golden("norm_replay")
    ns = O.NormStats(7)
    for s in range(5):
        O.norm_update(ns, g[f"n_x{s}"])
        np.testing.assert_allclose(ns.mean, g[f"n_mean{s}"], rtol=1e-14, atol=1e-14)
        np.testing.assert_allclose(ns.var, g[f"n_var{s}"], rtol=1e-14, atol=1e-14)
        assert ns.count == float(g[f"n_count{s}"])
        np.testing.assert_array_equal(O.norm_apply(ns, g[f"n_x{s}"]), g[f"n_apply{s}"])


def test_replay_ring_matches_reference(golden):
    g = golden("norm_replay")
    ring = O.Ring(37, O.codec_width(4, 2))
    for s in range(6):
        ring.insert(g[f"r_rows{s}"])
    assert tuple(ring.window()) == tuple(g["r_window"])
    idx = ring.sample_indices(64, O.philox_stream(1, "replay"))
    np.testing.assert_array_equal(idx, g["r_idx"])
    np.testing.assert_array_equal(ring.read(idx), g["r_read"])
    dec = O.codec_decode(4, 2, ring.read(idx))
    for k, v in dec.items():
        np.testing.assert_array_equal(v, g[f"r_dec_{k}"])
    with pytest.raises(IndexError):
        ring.read([0])
    # R:tests/test_replaypath.py ring eviction: cap 4, insert 3 then 6 -> window (5, 9)
    r = O.Ring(4, 1)
    r.insert(np.arange(3, dtype=np.float32)[:, None])
    r.insert(np.arange(3, 9, dtype=np.float32)[:, None])
    assert r.window() == (5, 9)
    np.testing.assert_array_equal(r.data[:, 0], [8, 5, 6, 7])


def test_perm_stream_matches_reference(golden):
    g = golden("perms")
    rng = O.philox_stream(1, "update")
    for e in range(3):
        np.testing.assert_array_equal(rng.permutation(96), g[f"perm{e}"])
    np.testing.assert_array_equal(O.philox_stream(1, "replay").integers(100, 1000, size=50),
                                  g["ints"])


# ------------------------------------------- LayerNorm: FD-pinned only (no ref)
def test_layernorm_oracle_fd():
    rng = np.random.default_rng(0)
    x = rng.normal(size=(3, 6))
    gam, bet = rng.normal(size=6), rng.normal(size=6)
    dy = rng.normal(size=(3, 6))
    _, cache = O.ln_forward(x, gam, bet)
    dx, dg, db = O.ln_backward(dy, gam, cache)
    h = 1e-6
    num = np.zeros_like(x)
    for i in range(x.shape[0]):
        for j in range(x.shape[1]):
            xp, xm = x.copy(), x.copy()
            xp[i, j] += h
            xm[i, j] -= h
            num[i, j] = ((O.ln_forward(xp, gam, bet)[0] * dy).sum()
                         - (O.ln_forward(xm, gam, bet)[0] * dy).sum()) / (2 * h)
    np.testing.assert_allclose(dx, num, atol=1e-6)
    np.testing.assert_allclose(db, dy.sum(0), atol=1e-12)
