"""GPU parity of the PPO / APPO learner (plan = K4 + K7 + K9 + K8 + K13)."""

import numpy as np
import pytest

from oracle import port as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2605_30313_b200 import algos as A  # noqa: E402
from paper_2605_30313_b200 import tensornet as TN  # noqa: E402
import paper_2605_30313_b200 as P  # noqa: E402


@pytest.fixture(autouse=True)
def fp32_mode():
    """The exact-fp32 parity configuration (SIMT GEMMs)."""
    old = P.get_precision()
    P.set_precision("fp32")
    yield
    P.set_precision(old)


def rel_err(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.abs(b))))


def _seg_kwargs(g, p):
    keys = ["obs", "critic_obs", "actions", "behavior_log_prob", "rewards", "terminated",
            "truncated", "values", "bootstrap_value", "truncation_values"]
    return {k: g[p + k] for k in keys}


def _ac(actor_dims, critic_dims, fa, fc):
    a = TN.ModelParams.from_numpy(TN.Arch(actor_dims[0], actor_dims[1:-1], actor_dims[-1]), fa)
    c = TN.ModelParams.from_numpy(TN.Arch(critic_dims[0], critic_dims[1:-1], critic_dims[-1]), fc)
    return A.AcParams(a, c)


def test_ppo_loss_and_grads_match_reference(golden):
    g = golden("ppo")
    seg = _seg_kwargs(g, "s_")
    params = _ac((10, 32, 16, 4), (12, 32, 16, 1), g["s_actor"], g["s_critic"])
    idx = g["s_idx"]
    adv = g["s_adv"].reshape(-1)
    advn = (adv - adv.mean()) / (adv.std() + 1e-8)
    flat = lambda a: a.reshape(-1, *a.shape[2:])
    terms, ga, gc = A.ppo_loss_and_grads(
        params, flat(seg["obs"])[idx], flat(seg["critic_obs"])[idx], flat(seg["actions"])[idx],
        seg["behavior_log_prob"].reshape(-1)[idx], advn[idx], g["s_ret"].reshape(-1)[idx],
        seg["values"].reshape(-1)[idx], A.PpoConfig())
    got = [terms[k] for k in ("policy_loss", "value_loss", "entropy", "total", "kl")]
    assert rel_err(got, g["s_terms"]) < 1e-5
    assert rel_err(ga.flat(), g["s_ga"]) < 1e-5
    assert rel_err(gc.flat(), g["s_gc"]) < 1e-5


def test_ppo_update_matches_reference(golden):
    """Full update on the reference's own permutation stream: parameters and
    stats within the fp32 full-update tolerance of SURVEY.md §8(c)."""
    from oracle.port import philox_stream

    g = golden("ppo")
    seg = A.RolloutSegment(**_seg_kwargs(g, "u_"))
    seg.advantages, seg.returns = A.gae(seg.rewards, seg.values, seg.terminated, seg.truncated,
                                        seg.bootstrap_value, 0.99, 0.95,
                                        truncation_values=seg.truncation_values)
    params = _ac((6, 16, 16, 3), (7, 16, 16, 1), g["u_actor0"], g["u_critic0"])
    cfg = A.PpoConfig(epochs=2, minibatches=4)
    opt = A.AcOpt.for_params(params, cfg.lr)
    st = A.ppo_update(seg, params, opt, cfg, philox_stream(1, "update"))
    d_ref = g["u_actor1"] - g["u_actor0"]
    d_gpu = params.actor.flat() - g["u_actor0"]
    assert np.linalg.norm(d_gpu - d_ref) / np.linalg.norm(d_ref) < 0.02
    np.testing.assert_allclose(params.actor.flat(), g["u_actor1"], atol=2e-5)
    np.testing.assert_allclose(params.critic.flat(), g["u_critic1"], atol=2e-5)
    got = [st.policy_loss, st.value_loss, st.entropy, st.kl, st.lr, st.grad_norm]
    assert rel_err(got, g["u_stats"]) < 1e-4
    assert opt.actor.t == 8 and opt.critic.t == 8


def test_ppo_update_divergence():
    rng = np.random.default_rng(8)
    t, b = 4, 3
    params = A.AcParams(TN.init_params(TN.Arch(3, (4,), 2), 7), TN.init_params(TN.Arch(4, (4,), 1), 8))
    seg = A.RolloutSegment(obs=rng.normal(size=(t, b, 3)).astype(np.float32),
                           critic_obs=rng.normal(size=(t, b, 4)).astype(np.float32),
                           actions=rng.normal(size=(t, b, 2)).astype(np.float32),
                           behavior_log_prob=rng.normal(size=(t, b)), rewards=rng.normal(size=(t, b)),
                           terminated=np.zeros((t, b), bool), truncated=np.zeros((t, b), bool),
                           values=rng.normal(size=(t, b)), bootstrap_value=rng.normal(size=b))
    opt = A.AcOpt.for_params(params, 1e-3)
    with pytest.raises(ValueError, match="advantages"):
        A.ppo_update(seg, params, opt, A.PpoConfig(), np.random.default_rng(0))
    seg.advantages = np.full((t, b), np.nan)
    seg.returns = np.zeros((t, b))
    before = params.actor.flat().copy()
    with pytest.raises(TN.DivergenceError):
        A.ppo_update(seg, params, opt, A.PpoConfig(minibatches=2), np.random.default_rng(0))
    np.testing.assert_array_equal(params.actor.flat(), before)
    seg.advantages = np.zeros((t, b))
    with pytest.raises(ValueError, match="divide"):
        A.ppo_update(seg, params, opt, A.PpoConfig(minibatches=5), np.random.default_rng(0))


from helpers import _synthetic  # noqa: E402


def test_ppo_single_step_cfg2_shape_vs_oracle_f64():
    """cfg2 shapes (obs 235, 512-256-128, mb 24576): one minibatch's grads vs
    the f64 oracle within 1e-5 x max(1, |ref|)."""
    T, N = 24, 1024  # 24,576 rows = one cfg2 minibatch
    seg, actor, critic = _synthetic(T, N, 235, 235, 12, (512, 256, 128), seed=3)
    adv, ret = O.gae(seg["rewards"], seg["values"], seg["terminated"], seg["truncated"],
                     seg["bootstrap_value"], 0.99, 0.95, seg["truncation_values"])
    advn = O.normalize_adv(adv.reshape(-1))
    to64 = lambda n: O.Net(n.dims, [[w.astype(np.float64), b.astype(np.float64)] for w, b in n.layers],
                           n.log_std.astype(np.float64))
    f = lambda a: a.reshape(-1, *a.shape[2:])
    args = (f(seg["obs"]).astype(np.float64), f(seg["critic_obs"]).astype(np.float64),
            f(seg["actions"]).astype(np.float64), seg["behavior_log_prob"].reshape(-1), advn,
            ret.reshape(-1), seg["values"].reshape(-1))
    terms, ga, gc = O.ppo_loss_grads(to64(actor), to64(critic), *args, O.PpoCfg())
    params = A.AcParams(TN.ModelParams.from_numpy(TN.Arch(235, (512, 256, 128), 12), actor.flat()),
                        TN.ModelParams.from_numpy(TN.Arch(235, (512, 256, 128), 1), critic.flat()))
    gterms, gga, ggc = A.ppo_loss_and_grads(params, f(seg["obs"]), f(seg["critic_obs"]),
                                            f(seg["actions"]), seg["behavior_log_prob"].reshape(-1),
                                            advn, ret.reshape(-1), seg["values"].reshape(-1),
                                            A.PpoConfig())
    for k in ("policy_loss", "value_loss", "entropy", "kl"):
        assert abs(gterms[k] - terms[k]) <= 1e-5 * max(1.0, abs(terms[k])), k
    assert rel_err(gga.flat(), ga.flat()) < 1e-5
    assert rel_err(ggc.flat(), gc.flat()) < 1e-5


def test_ppo_full_update_cfg1_vs_oracle():
    """cfg1 (1024 x 24, obs 48, 256-128-128, 5x4) full update: norm-based
    parameter-delta parity against the f32 oracle with the SAME permutations."""
    from oracle.port import philox_stream

    T, N = 24, 1024
    segd, actor, critic = _synthetic(T, N, 48, 48, 12, (256, 128, 128), seed=5)
    adv, ret = O.gae(segd["rewards"], segd["values"], segd["terminated"], segd["truncated"],
                     segd["bootstrap_value"], 0.99, 0.95, segd["truncation_values"])
    cfg = O.PpoCfg()
    a_ref, c_ref = actor.clone(), critic.clone()
    oa, oc = O.Opt.for_net(a_ref, cfg.lr), O.Opt.for_net(c_ref, cfg.lr)
    ref_seg = dict(segd, advantages=adv, returns=ret)
    ost = O.ppo_update(ref_seg, a_ref, c_ref, oa, oc, cfg, philox_stream(1, "update"))

    params = A.AcParams(TN.ModelParams.from_numpy(TN.Arch(48, (256, 128, 128), 12), actor.flat()),
                        TN.ModelParams.from_numpy(TN.Arch(48, (256, 128, 128), 1), critic.flat()))
    seg = A.RolloutSegment(**segd)
    seg.advantages, seg.returns = A.gae(seg.rewards, seg.values, seg.terminated, seg.truncated,
                                        seg.bootstrap_value, 0.99, 0.95,
                                        truncation_values=seg.truncation_values)
    opt = A.AcOpt.for_params(params, 1e-3)
    st = A.ppo_update(seg, params, opt, A.PpoConfig(), philox_stream(1, "update"))
    for ref_net, got, init in ((a_ref, params.actor, actor), (c_ref, params.critic, critic)):
        d_ref = ref_net.flat() - init.flat()
        d_gpu = got.flat() - init.flat()
        rel = np.linalg.norm(d_gpu - d_ref) / np.linalg.norm(d_ref)
        cos = float(d_gpu @ d_ref / (np.linalg.norm(d_gpu) * np.linalg.norm(d_ref)))
        assert rel <= 0.10 and cos >= 0.995, (rel, cos)
    assert abs(st.policy_loss - ost["policy_loss"]) < 1e-3
    assert abs(st.value_loss - ost["value_loss"]) <= 1e-3 * max(1, abs(ost["value_loss"]))
    assert abs(st.entropy - ost["entropy"]) < 1e-4


def test_appo_update_matches_reference(golden):
    """appo_update on the reference's goldens (behaviour policy perturbed by
    1e-2, V-trace rho/c clips 1, reference Philox permutations)."""
    from oracle.port import philox_stream

    g = golden("ppo")
    seg = A.RolloutSegment(**_seg_kwargs(g, "a_"), behavior_version=3)
    params = _ac((6, 16, 16, 3), (7, 16, 16, 1), g["a_actor0"], g["a_critic0"])
    cfg = A.AppoConfig(epochs=2, minibatches=2)
    opt = A.AcOpt.for_params(params, cfg.lr)
    st = A.appo_update(seg, params, opt, cfg, philox_stream(1, "update"), learner_version=5)
    np.testing.assert_allclose(params.actor.flat(), g["a_actor1"], atol=2e-5)
    np.testing.assert_allclose(params.critic.flat(), g["a_critic1"], atol=2e-5)
    got = [st.policy_loss, st.value_loss, st.entropy, st.kl, st.lr, st.grad_norm, st.staleness]
    assert rel_err(got, g["a_stats"]) < 1e-4


def test_learners_and_weight_slot():
    """PpoLearner / AppoLearner (runtime learner halves) + WeightSlot host snapshots."""
    import threading

    from paper_2605_30313_b200 import runtime as RT

    rng = np.random.default_rng(3)
    t, b, od, ad = 8, 32, 6, 2
    params = RT.build_ac_params(od, od, ad, (16, 16), seed=1)

    def segment(seq, version):
        return A.RolloutSegment(
            obs=rng.normal(size=(t, b, od)).astype(np.float32),
            critic_obs=rng.normal(size=(t, b, od)).astype(np.float32),
            actions=rng.normal(size=(t, b, ad)).astype(np.float32),
            behavior_log_prob=rng.normal(size=(t, b)) - 3.0, rewards=rng.normal(size=(t, b)),
            terminated=rng.random((t, b)) < 0.05, truncated=np.zeros((t, b), bool),
            values=rng.normal(size=(t, b)), bootstrap_value=rng.normal(size=b),
            truncation_values=np.zeros((t, b)), behavior_version=version, seq=seq)

    learner = RT.PpoLearner(params, A.PpoConfig(epochs=1, minibatches=2), A.DeviceRng(0))
    learner.slot.publish(params)
    v0, snap0 = learner.slot.fetch()
    st = learner.learn(segment(0, v0), 0)
    assert np.isfinite(st.policy_loss)
    v1, snap1 = learner.slot.fetch()
    assert v1 == v0 + 1
    np.testing.assert_array_equal(snap1.actor.flat(), params.actor.flat())
    assert not np.array_equal(snap0.actor.flat(), snap1.actor.flat())
    with pytest.raises(ValueError):
        snap1.actor.layers[0][0][0, 0] = 1.0  # published snapshots are frozen

    appo = RT.AppoLearner(params, A.AppoConfig(epochs=1, minibatches=2), A.DeviceRng(1))
    appo.slot.publish(params)
    ring = RT.RolloutRing(2)

    def produce():
        for s in range(4):
            ring.put(segment(s, appo.slot.version))

    th = threading.Thread(target=produce)
    th.start()
    stats = appo.drain(ring, 4)
    th.join()
    assert len(stats) == 4 and max(appo.staleness) <= 2 + 1


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_pipeline_matches_serial_updates(prec):
    """PpoPipeline (double-buffered H2D ring, device GAE) == host gae +
    ppo_update on the same segments and device permutation stream."""
    old = P.get_precision()
    P.set_precision(prec)
    try:
        T, N = 8, 512
        segs = []
        for sd in (3, 4, 5):
            segd, actor, critic = _synthetic(T, N, 48, 52, 12, (128, 64), seed=sd)
            segs.append(A.RolloutSegment(**segd))
        cfg = A.PpoConfig(epochs=2, minibatches=2)
        arch_a, arch_c = TN.Arch(48, (128, 64), 12), TN.Arch(52, (128, 64), 1)

        def fresh():
            p = A.AcParams(TN.ModelParams.from_numpy(arch_a, actor.flat()),
                           TN.ModelParams.from_numpy(arch_c, critic.flat()))
            return p, A.AcOpt.for_params(p, cfg.lr)

        p1, o1 = fresh()
        rng1 = A.DeviceRng(7)
        serial = []
        for sg in segs:
            sg.advantages, sg.returns = A.gae(sg.rewards, sg.values, sg.terminated, sg.truncated,
                                              sg.bootstrap_value, cfg.gamma, cfg.lam,
                                              truncation_values=sg.truncation_values)
            serial.append(A.ppo_update(sg, p1, o1, cfg, rng1))
        p2, o2 = fresh()
        pipe = A.PpoPipeline(p2, o2, cfg, A.DeviceRng(7))
        pipe.prefetch(segs[0])
        piped = []
        for i in range(len(segs)):
            piped.append(pipe.update(next_segment=segs[i + 1] if i + 1 < len(segs) else None))
        for a, b in zip(serial, piped):
            assert a.policy_loss == b.policy_loss and a.value_loss == b.value_loss
        np.testing.assert_array_equal(p1.actor.flat(), p2.actor.flat())
        np.testing.assert_array_equal(p1.critic.flat(), p2.critic.flat())
    finally:
        P.set_precision(old)


def _pipe_setup(nseg, T=8, N=512):
    segs = []
    for sd in range(3, 3 + nseg):
        segd, actor, critic = _synthetic(T, N, 48, 52, 12, (128, 64), seed=sd)
        segs.append(A.RolloutSegment(**segd))
    cfg = A.PpoConfig(epochs=2, minibatches=2)
    arch_a, arch_c = TN.Arch(48, (128, 64), 12), TN.Arch(52, (128, 64), 1)

    def fresh():
        p = A.AcParams(TN.ModelParams.from_numpy(arch_a, actor.flat()),
                       TN.ModelParams.from_numpy(arch_c, critic.flat()))
        return p, A.AcOpt.for_params(p, cfg.lr)

    return segs, cfg, fresh


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_pipeline_async_chained_matches_serial(prec):
    """update_async: update i+1 enqueued (Adam step counters continued on the
    device) before update i's statistics are read == serial updates, bit for
    bit, and the host step counters end where the serial run's do."""
    old = P.get_precision()
    P.set_precision(prec)
    try:
        segs, cfg, fresh = _pipe_setup(4)
        p1, o1 = fresh()
        rng1 = A.DeviceRng(7)
        serial = []
        for sg in segs:
            sg.advantages, sg.returns = A.gae(sg.rewards, sg.values, sg.terminated, sg.truncated,
                                              sg.bootstrap_value, cfg.gamma, cfg.lam,
                                              truncation_values=sg.truncation_values)
            serial.append(A.ppo_update(sg, p1, o1, cfg, rng1))
        p2, o2 = fresh()
        pipe = A.PpoPipeline(p2, o2, cfg, A.DeviceRng(7))
        pipe.prefetch(segs[0])
        hs, piped = [], []
        for i in range(len(segs)):
            hs.append(pipe.update_async(next_segment=segs[i + 1] if i + 1 < len(segs) else None))
            if i >= 1:
                piped.append(hs[i - 1].result())
        piped.append(hs[-1].result())
        for a, b in zip(serial, piped):
            assert a.policy_loss == b.policy_loss and a.value_loss == b.value_loss
            assert a.grad_norm == b.grad_norm and a.kl == b.kl
        np.testing.assert_array_equal(p1.actor.flat(), p2.actor.flat())
        np.testing.assert_array_equal(p1.critic.flat(), p2.critic.flat())
        assert (o2.actor.t, o2.critic.t) == (o1.actor.t, o1.critic.t)
        # a plain update() after the chain starts from the device-chained state
        pipe.prefetch(segs[0])
        b = pipe.update()
        a = A.ppo_update(segs[0], p1, o1, cfg, rng1)
        assert a.policy_loss == b.policy_loss
        np.testing.assert_array_equal(p1.actor.flat(), p2.actor.flat())
    finally:
        P.set_precision(old)


def test_pipeline_async_divergence_latch_carries():
    """A diverging update inside a chain: its result raises DivergenceError,
    and the update already queued behind it inherits the latch on the device
    (no step applied), so the parameters stay where the last good update
    left them -- as after the serial reference's DivergenceError."""
    segs, cfg, fresh = _pipe_setup(3, T=6, N=256)
    segs[1].rewards[0, 0] = np.nan
    p1, o1 = fresh()
    sg = segs[0]
    sg.advantages, sg.returns = A.gae(sg.rewards, sg.values, sg.terminated, sg.truncated,
                                      sg.bootstrap_value, cfg.gamma, cfg.lam,
                                      truncation_values=sg.truncation_values)
    A.ppo_update(sg, p1, o1, cfg, A.DeviceRng(9))
    p2, o2 = fresh()
    pipe = A.PpoPipeline(p2, o2, cfg, A.DeviceRng(9))
    pipe.prefetch(segs[0])
    h0 = pipe.update_async(next_segment=segs[1])
    h1 = pipe.update_async(next_segment=segs[2])
    h2 = pipe.update_async()
    h0.result()
    with pytest.raises(TN.DivergenceError):
        h1.result()
    with pytest.raises(TN.DivergenceError):
        h2.result()
    np.testing.assert_array_equal(p1.actor.flat(), p2.actor.flat())
    np.testing.assert_array_equal(p1.critic.flat(), p2.critic.flat())


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_ppo_data_parallel_two_ranks_match_single_process(prec):
    """SURVEY.md 8(e) for PPO: two ranks (threads on one GPU; the all-reduce a
    barrier + sum) in replicated-segment mode each take half of every
    reference-permuted minibatch; after the per-step gradient all-reduce the
    replicated clip + Adam reproduce the single-process update (fp32: to
    3e-6; bf16 -- fused output stage, batched dW -- to the bf16 bound), and the
    ranks' parameters are bit-identical either way."""
    import threading

    from oracle.port import philox_stream
    from paper_2605_30313_b200 import _dist

    old = P.get_precision()
    P.set_precision(prec)
    try:
        T, N = 8, 256
        segd, actor, critic = _synthetic(T, N, 48, 52, 12, (128, 64), seed=11)
        cfg = A.PpoConfig(epochs=2, minibatches=2)
        arch_a, arch_c = TN.Arch(48, (128, 64), 12), TN.Arch(52, (128, 64), 1)

        def fresh():
            p = A.AcParams(TN.ModelParams.from_numpy(arch_a, actor.flat()),
                           TN.ModelParams.from_numpy(arch_c, critic.flat()))
            return p, A.AcOpt.for_params(p, cfg.lr)

        def seg():
            s = A.RolloutSegment(**segd)
            s.advantages, s.returns = A.gae(s.rewards, s.values, s.terminated, s.truncated,
                                            s.bootstrap_value, cfg.gamma, cfg.lam,
                                            truncation_values=s.truncation_values)
            return s

        p_ref, o_ref = fresh()
        want = A.ppo_update(seg(), p_ref, o_ref, cfg, philox_stream(1, "update"))

        class Reducer:
            def __init__(self):
                self.bar = threading.Barrier(2)
                self.slots = {}

            def __call__(self, rank, t):
                self.slots[rank] = t
                torch.cuda.synchronize()
                self.bar.wait()
                if rank == 0:
                    total = self.slots[0] + self.slots[1]
                    self.slots[0].copy_(total)
                    self.slots[1].copy_(total)
                    torch.cuda.synchronize()
                self.bar.wait()

        red = Reducer()
        got = [None, None]
        errors = []
        segs = [seg(), seg()]
        states = [fresh(), fresh()]

        def run(rank):
            try:
                _dist.emulate_rank(2, rank, lambda t: red(rank, t))
                p, o = states[rank]
                got[rank] = A.ppo_update(segs[rank], p, o, cfg, philox_stream(1, "update"))
            except Exception as e:  # pragma: no cover
                errors.append(e)
                red.bar.abort()
            finally:
                _dist.clear_emulation()

        th = [threading.Thread(target=run, args=(r,)) for r in range(2)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        assert not errors, errors
        np.testing.assert_array_equal(states[0][0].actor.flat(), states[1][0].actor.flat())
        np.testing.assert_array_equal(states[0][0].critic.flat(), states[1][0].critic.flat())
        if prec == "fp32":
            for p, _ in states:
                np.testing.assert_allclose(p.actor.flat(), p_ref.actor.flat(), atol=3e-6)
                np.testing.assert_allclose(p.critic.flat(), p_ref.critic.flat(), atol=3e-6)
            for g in got:
                assert g.policy_loss == pytest.approx(want.policy_loss, abs=1e-5)
                assert g.value_loss == pytest.approx(want.value_loss, rel=1e-5, abs=1e-6)
        else:
            a0, c0 = actor.flat(), critic.flat()
            for p, _ in states:
                for got_p, ref_p, init in ((p.actor.flat(), p_ref.actor.flat(), a0),
                                           (p.critic.flat(), p_ref.critic.flat(), c0)):
                    d_ref, d_got = ref_p - init, got_p - init
                    cos = float(d_got @ d_ref / (np.linalg.norm(d_got) * np.linalg.norm(d_ref)))
                    assert cos >= 0.97, cos
            for g in got:
                assert g.policy_loss == pytest.approx(want.policy_loss, abs=1e-2)
                assert g.value_loss == pytest.approx(want.value_loss, rel=1e-2, abs=1e-2)
    finally:
        P.set_precision(old)


def test_pipeline_per_step_streaming_matches_prefetch():
    """Per-step segment streaming stages exactly the
    bytes a whole-segment prefetch does: identical update results."""
    T, N = 6, 256
    segd, actor, critic = _synthetic(T, N, 40, 44, 6, (64, 64), seed=21)
    cfg = A.PpoConfig(epochs=2, minibatches=2)
    arch_a, arch_c = TN.Arch(40, (64, 64), 6), TN.Arch(44, (64, 64), 1)

    def run(stream):
        p = A.AcParams(TN.ModelParams.from_numpy(arch_a, actor.flat()),
                       TN.ModelParams.from_numpy(arch_c, critic.flat()))
        pipe = A.PpoPipeline(p, A.AcOpt.for_params(p, cfg.lr), cfg, A.DeviceRng(5))
        seg = A.RolloutSegment(**segd)
        if stream:
            w = pipe.stream_segment(T, N)
            for t in range(T):
                w.push(t, seg.obs[t], seg.critic_obs[t], seg.actions[t],
                       seg.behavior_log_prob[t], seg.rewards[t], seg.terminated[t],
                       seg.truncated[t], seg.values[t],
                       None if seg.truncation_values is None else seg.truncation_values[t])
            w.finish(seg.bootstrap_value)
        else:
            pipe.prefetch(seg)
        st = pipe.update()
        return st, p

    s1, p1 = run(False)
    s2, p2 = run(True)
    assert s1.policy_loss == s2.policy_loss and s1.value_loss == s2.value_loss
    np.testing.assert_array_equal(p1.actor.flat(), p2.actor.flat())
    np.testing.assert_array_equal(p1.critic.flat(), p2.critic.flat())


def test_checkpoint_roundtrip_and_reference_format(tmp_path):
    """save/load_checkpoint (R:tensornet/checkpoint.py:23-81): device params +
    normalizer round-trip, and the npz keys/shapes the reference reads."""
    arch = TN.Arch(7, (16, 8), 3)
    p = TN.init_params(arch, 4)
    p.version = 9
    norm = TN.Normalizer(7, count=5.0, mean=np.arange(7.0), var=np.ones(7) * 2.0, frozen=True)
    path = tmp_path / "ck.npz"
    TN.save_checkpoint(path, p, norm)
    with np.load(path) as d:
        assert d["layer0_w"].shape == (16, 7) and d["layer2_b"].shape == (3,)
        assert int(d["version"]) == 9 and d["log_std"].shape == (3,)
    q, n2 = TN.load_checkpoint(path)
    np.testing.assert_array_equal(q.flat(), p.flat())
    assert q.version == 9 and q.arch == arch
    np.testing.assert_array_equal(n2.mean, np.arange(7.0))
    assert n2.count == 5.0 and n2.frozen


def test_checkpoint_reads_reference_file():
    """A checkpoint written by the reference's own save_checkpoint
    (tests/golden/gen_checkpoint.py) loads into device params unchanged."""
    from pathlib import Path

    g = Path(__file__).resolve().parent / "golden"
    q, n = TN.load_checkpoint(g / "ckpt_ref.npz")
    e = np.load(g / "ckpt_ref_expect.npz")
    np.testing.assert_array_equal(q.flat(), e["flat"])
    assert q.version == 17 and q.arch.hidden_dims == (8, 4)
    np.testing.assert_allclose(n.mean, e["mean"], rtol=0, atol=0)
    np.testing.assert_allclose(n.var, e["var"], rtol=0, atol=0)
    assert n.count == float(e["count"])


def test_gpu_trace_spans_on_host_clock():
    """Tracer.gpu_span: CUDA-event spans converted to the host clock, ordered,
    with device durations."""
    from paper_2605_30313_b200.trace import Tracer

    tr = Tracer()
    x = torch.randn(4096, 4096, device="cuda")
    with tr.gpu_span("learner", "learner/update"):
        for _ in range(4):
            x = x @ x * 1e-3
    with tr.gpu_span("learner", "learner/replay_sample"):
        x.add_(1.0)
    assert tr.flush_gpu() == 2
    ev = tr.events()
    assert [e.name for e in ev] == ["learner/update", "learner/replay_sample"]
    assert ev[0].duration_ns > 0 and ev[1].ts_start >= ev[0].ts_start


def test_weight_slot_snapshot_never_mixes_versions():
    """R:runtime/sync.py:40-54 'never a mix': an in-place parameter write queued
    right behind a non-blocking publish must not leak into the snapshot (the
    publish snapshots on the learner stream before the slow D2H)."""
    from paper_2605_30313_b200 import runtime as RT

    p = TN.init_params(TN.Arch(256, (1024, 1024), 64), 0)  # ~1.4M params
    want = p.flat().astype(np.float32)
    slot = RT.WeightSlot()
    for k in range(3):
        slot.publish(p)
        p.buf.add_(1.0)  # the next "update", in place, on the learner stream
        v, snap = slot.fetch()
        assert v == k + 1
        np.testing.assert_array_equal(snap.flat(), want)
        want = want + np.float32(1.0)
