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
