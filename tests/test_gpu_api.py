"""The reference's per-call SAC / Gaussian-head API on the device, against
golden vectors written by the UNMODIFIED reference (tests/golden/gen_api.py):
gaussian_dist (plain / squashed, sample / evaluate), squashed_log_prob,
sample_squashed (R:tensornet/distributions.py:29-84) and critic_target,
critic_loss_and_grads, actor_loss_and_grads, alpha_loss_and_grad
(R:algos/sac.py:111-229).  fp32 (exact) GEMM back end; bound 1e-5 relative
(max(1, |ref|) floor)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2605_30313_b200 as P  # noqa: E402
from paper_2605_30313_b200 import algos as A  # noqa: E402
from paper_2605_30313_b200 import tensornet as TN  # noqa: E402
from paper_2605_30313_b200.algos import sac as S  # noqa: E402


@pytest.fixture(autouse=True)
def fp32_mode():
    old = P.get_precision()
    P.set_precision("fp32")
    yield
    P.set_precision(old)


def _rel(got, ref):
    got = np.asarray(got.cpu().numpy() if isinstance(got, torch.Tensor) else got, np.float64)
    ref = np.asarray(ref, np.float64)
    assert got.shape == ref.shape, (got.shape, ref.shape)
    return float(np.max(np.abs(got - ref) / np.maximum(1.0, np.abs(ref))))


def _philox(seed, label):
    from oracle.port import philox_stream

    return philox_stream(seed, label)


@pytest.mark.parametrize("mode", [0, 1, 2, 3])
def test_gaussian_dist_matches_reference(golden, mode):
    g = golden("api")
    action = g["g_act"] if mode in (1, 3) else None
    s, lp, ent = TN.gaussian_dist(g["g_mean"], g["g_log_std"], action=action,
                                  squashed=mode >= 2, rng=_philox(4, f"dist{mode}"))
    assert _rel(s, g[f"g{mode}_sample"]) < 1e-12
    assert _rel(lp, g[f"g{mode}_logp"]) < 1e-10
    assert _rel(ent, g[f"g{mode}_ent"]) < 1e-12


def test_squashed_log_prob_and_sample_squashed_match_reference(golden):
    g = golden("api")
    lp = TN.squashed_log_prob(g["g_mean"], g["g_log_std"], g["g_u"], np.tanh(g["g_u"]))
    assert _rel(lp, g["g_sqlp"]) < 1e-10
    a, u, logp = TN.sample_squashed(g["g_mean"].astype(np.float32),
                                    g["g_log_std"].astype(np.float32), g["s_eps"])
    assert _rel(u, g["s_u"]) < 1e-6  # same f32 op order (expf may differ by an ulp)
    assert _rel(a, g["s_a"]) < 1e-6
    # float32 log1p(-a^2 + 1e-6) near |a| = 1 turns one-ulp tanhf differences
    # into ~1e-4 absolute log-prob differences (the reference is float32 too)
    assert _rel(logp, g["s_logp"]) < 1e-3


def _params(g):
    od, ad = g["b_obs"].shape[1], g["b_action"].shape[1]
    qa = TN.Arch(od + ad, (64, 32), 1)
    mk = TN.ModelParams.from_numpy
    return A.SacParams(actor=mk(TN.Arch(od, (64, 32), ad), g["p_actor"]), q1=mk(qa, g["p_q1"]),
                       q2=mk(qa, g["p_q2"]), q1_targ=mk(qa, g["p_q1t"]),
                       q2_targ=mk(qa, g["p_q2t"]), log_alpha=float(g["p_log_alpha"]))


def _batch(g):
    return {k: g[f"b_{k}"] for k in ("obs", "action", "reward", "next_obs", "terminated",
                                     "n_used")}


def test_critic_target_matches_reference(golden):
    g = golden("api")
    y = S.critic_target(_params(g), _batch(g), A.SacConfig().gamma, _philox(1, "learner"))
    assert y.dtype == torch.float64
    assert _rel(y, g["y"]) < 1e-5


def test_critic_loss_and_grads_matches_reference(golden):
    g = golden("api")
    b = _batch(g)
    q_in = np.concatenate([b["obs"], b["action"]], axis=-1)
    loss, grads, pred = S.critic_loss_and_grads(_params(g).q1, q_in, g["y"])
    assert _rel(loss, g["c_loss"]) < 1e-5
    assert _rel(pred, g["c_pred"]) < 1e-5
    assert _rel(grads.flat(), g["c_grads"]) < 1e-5


def test_actor_and_alpha_loss_match_reference(golden):
    g = golden("api")
    loss, grads, logp = S.actor_loss_and_grads(_params(g), g["b_obs"], g["a_eps"])
    assert _rel(loss, g["a_loss"]) < 1e-5
    # (f32 log1p(1 - a^2 + 1e-6) amplifies a one-ulp tanhf difference near |a| = 1)
    assert _rel(logp, g["a_logp"]) < 1e-4
    assert _rel(grads.flat(), g["a_grads"]) < 1e-5
    al, dla = S.alpha_loss_and_grad(float(g["p_log_alpha"]), logp, -1.5)
    assert _rel([al, dla], g["al"]) < 1e-5
