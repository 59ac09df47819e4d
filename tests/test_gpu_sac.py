"""GPU parity of the SAC plan (K10 target, K11 heads, K12 Polyak, K13 Adam,
alpha ScalarAdam) against the reference's own sac_update trajectory."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2605_30313_b200 as P  # noqa: E402
from paper_2605_30313_b200 import algos as A  # noqa: E402
from paper_2605_30313_b200 import tensornet as TN  # noqa: E402


@pytest.fixture(autouse=True)
def fp32_mode():
    old = P.get_precision()
    P.set_precision("fp32")
    yield
    P.set_precision(old)


def _state(g, cfg):
    od, ad = 5, 2
    actor = TN.ModelParams.from_numpy(TN.Arch(od, (16, 16), ad), g["actor0"])
    q1 = TN.ModelParams.from_numpy(TN.Arch(od + ad, (16, 16), 1), g["q10"])
    q2 = TN.ModelParams.from_numpy(TN.Arch(od + ad, (16, 16), 1), g["q20"])
    return A.SacState.create(actor, q1, q2, cfg)


def test_sac_updates_match_reference(golden):
    """Four sac_update calls (policy_frequency 2: two actor/alpha steps) on the
    reference's learner noise stream: losses, alpha and all five parameter
    sets track the reference trajectory."""
    from oracle.port import philox_stream

    g = golden("sac")
    cfg = A.SacConfig(policy_frequency=2, batch_size=16)
    st = _state(g, cfg)
    rng = philox_stream(1, "learner")
    for s in range(4):
        batch = {k: g[f"b{s}_{k}"] for k in ("obs", "action", "reward", "next_obs",
                                             "terminated", "n_used")}
        out = A.sac_update(batch, st, cfg, rng)
        ref = g[f"stats{s}"]
        got = np.array([out.extra.get(k, np.nan) for k in ("critic_loss", "actor_loss",
                                                           "alpha_loss", "alpha")])
        np.testing.assert_allclose(got, ref, rtol=1e-4, atol=1e-6)
        p = st.params
        for name, net in (("actor", p.actor), ("q1", p.q1), ("q2", p.q2), ("q1t", p.q1_targ),
                          ("q2t", p.q2_targ)):
            np.testing.assert_allclose(net.flat(), g[f"{name}{s + 1}"], atol=2e-5, err_msg=name)
        assert p.log_alpha == pytest.approx(float(g[f"log_alpha{s + 1}"]), abs=1e-7)
    assert st.update_count == 4 and st.actor_opt.t == 2 and st.q1_opt.t == 4


def test_sac_rejects_tiny_batch(golden):
    g = golden("sac")
    cfg = A.SacConfig()
    st = _state(g, cfg)
    batch = {k: g[f"b0_{k}"][:1] for k in ("obs", "action", "reward", "next_obs", "terminated",
                                           "n_used")}
    with pytest.raises(ValueError, match="at least 2"):
        A.sac_update(batch, st, cfg, np.random.default_rng(0))


def test_soft_update_known_answer():
    t = TN.init_params(TN.Arch(3, (4,), 1), 0)
    o = TN.init_params(TN.Arch(3, (4,), 1), 1)
    t.buf.zero_()
    o.buf.fill_(1.0)
    A.soft_update(t, o, 0.125)
    assert float(t.buf[0].item()) == pytest.approx(0.125)


def test_sac_data_parallel_two_ranks_match_single_process(golden):
    """SURVEY.md 8(e) for SAC: two data-parallel ranks (emulated as threads on
    one GPU, the all-reduce a barrier + sum) each update on half of the batch
    with the global-batch loss scaling; after all-reducing the critic and
    actor gradients (+ loss / log-pi sums) the replicated Adam / alpha /
    Polyak steps reproduce the single-process trajectory on the whole batch."""
    import threading

    from oracle.port import philox_stream
    from paper_2605_30313_b200 import _dist

    g = golden("sac")
    cfg = A.SacConfig(policy_frequency=2, batch_size=16)
    ref = _state(g, cfg)
    ranks = [_state(g, cfg), _state(g, cfg)]
    rng_ref = philox_stream(1, "learner")
    rngs = [philox_stream(1, "learner"), philox_stream(1, "learner")]

    class Reducer:
        def __init__(self):
            self.bar = threading.Barrier(2)
            self.slots = {}

        def __call__(self, rank, t):
            self.slots[rank] = t
            self.bar.wait()
            if rank == 0:
                total = self.slots[0] + self.slots[1]
                self.slots[0].copy_(total)
                self.slots[1].copy_(total)
            torch.cuda.synchronize()
            self.bar.wait()

    red = Reducer()
    outs = [None, None]
    errors = []

    def run(rank, batch):
        try:
            _dist.emulate_rank(2, rank, lambda t: red(rank, t))
            outs[rank] = A.sac_update(batch, ranks[rank], cfg, rngs[rank])
        except Exception as e:  # pragma: no cover - surfaced below
            errors.append(e)
            red.bar.abort()
        finally:
            _dist.clear_emulation()

    for s in range(4):
        batch = {k: g[f"b{s}_{k}"] for k in ("obs", "action", "reward", "next_obs",
                                             "terminated", "n_used")}
        want = A.sac_update(batch, ref, cfg, rng_ref)
        th = [threading.Thread(target=run, args=(r, batch)) for r in range(2)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        assert not errors, errors
        for k in ("critic_loss", "actor_loss", "alpha_loss", "alpha"):
            if k in want.extra:
                for o in outs:
                    assert o.extra[k] == pytest.approx(want.extra[k], rel=1e-5, abs=1e-6), k
        for st in ranks:
            for a, b in ((st.params.actor, ref.params.actor), (st.params.q1, ref.params.q1),
                         (st.params.q2_targ, ref.params.q2_targ)):
                np.testing.assert_allclose(a.flat(), b.flat(), atol=2e-6)
            assert st.params.log_alpha == pytest.approx(ref.params.log_alpha, abs=1e-9)
        np.testing.assert_array_equal(ranks[0].params.q1.flat(), ranks[1].params.q1.flat())


@pytest.mark.parametrize("prec,tol,patol", [("fp32", 3e-5, 2e-5), ("bf16", 2e-2, 3e-3)])
def test_sac_layernorm_critics_match_oracle(prec, tol, patol):
    """cfg3's FastSAC critics carry LayerNorm (extension; the oracle's LN is
    FD-pinned): four updates with LN twin critics track the oracle's
    LN-extended sac_update (losses, and every parameter set incl. g / beta)."""
    from oracle import port as O

    P.set_precision(prec)
    od, ad, hid, n = 12, 4, (64, 32), 256
    rng = np.random.default_rng(3)
    a0 = O.net_init((od, *hid, ad), 0)
    q0 = [O.net_init((od + ad, *hid, 1), s, layer_norm=True) for s in (1, 2)]
    for q in q0:  # non-trivial gains / shifts
        for g, b in q.ln:
            g[:] = rng.uniform(0.5, 1.5, g.shape)
            b[:] = rng.normal(0, 0.2, b.shape)
    ocfg = O.SacCfg(policy_frequency=2)
    ost = O.SacSt.create(a0.clone(), q0[0].clone(), q0[1].clone(), ocfg)
    cfg = A.SacConfig(policy_frequency=2, batch_size=n)
    qa = TN.Arch(od + ad, hid, 1, layer_norm=True)
    st = A.SacState.create(TN.ModelParams.from_numpy(TN.Arch(od, hid, ad), a0.flat()),
                           TN.ModelParams.from_numpy(qa, q0[0].flat()),
                           TN.ModelParams.from_numpy(qa, q0[1].flat()), cfg)
    r_ref, r_got = O.philox_stream(5, "learner"), O.philox_stream(5, "learner")
    for s in range(4):
        batch = dict(obs=rng.normal(size=(n, od)).astype(np.float32),
                     action=np.tanh(rng.normal(size=(n, ad))).astype(np.float32),
                     reward=rng.normal(size=n).astype(np.float32),
                     next_obs=rng.normal(size=(n, od)).astype(np.float32),
                     terminated=rng.random(n) < 0.05, n_used=np.ones(n, np.int64))
        want = O.sac_update(batch, ost, ocfg, r_ref)
        got = A.sac_update(batch, st, cfg, r_got).extra
        for k in want:
            assert got[k] == pytest.approx(want[k], rel=tol, abs=tol * 1e-1), (s, k)
        p = st.params
        for mine, ref in ((p.actor, ost.actor), (p.q1, ost.q1), (p.q2, ost.q2),
                          (p.q1_targ, ost.q1t), (p.q2_targ, ost.q2t)):
            # patol: bf16 activations may flip the sign of near-zero Adam
            # steps (|step| <= lr = 3e-4 per update)
            d = np.abs(mine.flat() - ref.flat()).max()
            assert d < patol, (s, d)
