"""3xTF32 (``set_precision("tf32x3")``): the exact-fp32 parity contract of
SURVEY.md 8(c) on the tcgen05 tensor cores.  Every MLP GEMM runs as ONE
kind::tf32 GEMM over a tripled K of split operands (A' = [A_hi | A_hi | A_lo],
B' = [B_hi | B_lo | B_hi]: hi*hi + hi*lo + lo*hi, csrc/gemm_tc.cu) with the
fp32 path's epilogues.  Bounds are the fp32 ones: 1e-5 x max(1, |ref|)
against the float64 oracle for one pass / one minibatch step; the reference's
own float32 trajectory for whole updates."""

import numpy as np
import pytest

from oracle import port as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2605_30313_b200 as P  # noqa: E402
from paper_2605_30313_b200 import algos as A  # noqa: E402
from paper_2605_30313_b200 import tensornet as TN  # noqa: E402
from helpers import _synthetic  # noqa: E402


@pytest.fixture(autouse=True)
def x3_mode():
    old = P.get_precision()
    P.set_precision("tf32x3")
    yield
    P.set_precision(old)


def _rel(got, ref):
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    return float(np.max(np.abs(got - ref) / np.maximum(1.0, np.abs(ref))))


def _to64(n):
    return O.Net(n.dims, [[w.astype(np.float64), b.astype(np.float64)] for w, b in n.layers],
                 n.log_std.astype(np.float64))


@pytest.mark.parametrize("M,dims", [(4096, (235, 512, 256, 128, 12)), (777, (48, 256, 128, 1))])
def test_mlp_forward_backward_x3_vs_f64(M, dims):
    rng = np.random.default_rng(M)
    net = O.net_init(dims, 3)
    x = rng.normal(size=(M, dims[0])).astype(np.float32)
    dout = (rng.normal(size=(M, dims[-1])) / M).astype(np.float32)
    y64, acts = O.mlp_forward(_to64(net), x.astype(np.float64))
    dx64, g64 = O.mlp_backward(_to64(net), x.astype(np.float64), acts, dout.astype(np.float64))
    p = TN.ModelParams.from_numpy(TN.Arch(dims[0], dims[1:-1], dims[-1]), net.flat())
    y, cache = TN.forward(p, x)
    dx, gr = TN.backward(p, cache, dout)
    assert _rel(y.cpu().numpy(), y64) < 1e-5
    assert _rel(dx.cpu().numpy(), dx64) < 1e-5
    assert _rel(gr.flat(), g64.flat()) < 1e-5


def test_ppo_single_step_cfg2_x3_vs_f64():
    """One cfg2 minibatch (24,576 rows, obs 235, 512-256-128): losses and both
    networks' gradients within 1e-5 x max(1, |ref|) of the float64 oracle."""
    T, N = 24, 1024
    seg, actor, critic = _synthetic(T, N, 235, 235, 12, (512, 256, 128), seed=3)
    adv, ret = O.gae(seg["rewards"], seg["values"], seg["terminated"], seg["truncated"],
                     seg["bootstrap_value"], 0.99, 0.95, seg["truncation_values"])
    advn = O.normalize_adv(adv.reshape(-1))
    f = lambda a: a.reshape(-1, *a.shape[2:])  # noqa: E731
    args = (f(seg["obs"]).astype(np.float64), f(seg["critic_obs"]).astype(np.float64),
            f(seg["actions"]).astype(np.float64), seg["behavior_log_prob"].reshape(-1), advn,
            ret.reshape(-1), seg["values"].reshape(-1))
    terms, ga, gc = O.ppo_loss_grads(_to64(actor), _to64(critic), *args, O.PpoCfg())
    params = A.AcParams(TN.ModelParams.from_numpy(TN.Arch(235, (512, 256, 128), 12), actor.flat()),
                        TN.ModelParams.from_numpy(TN.Arch(235, (512, 256, 128), 1), critic.flat()))
    gterms, gga, ggc = A.ppo_loss_and_grads(params, f(seg["obs"]), f(seg["critic_obs"]),
                                            f(seg["actions"]), seg["behavior_log_prob"].reshape(-1),
                                            advn, ret.reshape(-1), seg["values"].reshape(-1),
                                            A.PpoConfig())
    for k in ("policy_loss", "value_loss", "entropy", "kl"):
        assert abs(gterms[k] - terms[k]) <= 1e-5 * max(1.0, abs(terms[k])), k
    assert _rel(gga.flat(), ga.flat()) < 1e-5
    assert _rel(ggc.flat(), gc.flat()) < 1e-5


def test_ppo_cfg2_full_update_x3_tracks_f32_reference():
    """The benchmarked update (24 x 4096, 5 x 4, reference permutation stream)
    tracks the reference's own float32 update as closely as the SIMT fp32 path
    (<= 0.05 / >= 0.999; the SIMT path measures 0.009 / 0.99996)."""
    from threadpoolctl import threadpool_limits

    T, N, od, ad, hid = 24, 4096, 235, 12, (512, 256, 128)
    segd, actor, critic = _synthetic(T, N, od, od, ad, hid, seed=9)
    adv, ret = O.gae(segd["rewards"], segd["values"], segd["terminated"], segd["truncated"],
                     segd["bootstrap_value"], 0.99, 0.95, segd["truncation_values"])
    cfg = O.PpoCfg()
    a_ref, c_ref = actor.clone(), critic.clone()
    with threadpool_limits(limits=None):
        ost = O.ppo_update(dict(segd, advantages=adv, returns=ret), a_ref, c_ref,
                           O.Opt.for_net(a_ref, cfg.lr), O.Opt.for_net(c_ref, cfg.lr), cfg,
                           O.philox_stream(1, "update"))
    params = A.AcParams(TN.ModelParams.from_numpy(TN.Arch(od, hid, ad), actor.flat()),
                        TN.ModelParams.from_numpy(TN.Arch(od, hid, 1), critic.flat()))
    seg = A.RolloutSegment(**segd)
    seg.advantages, seg.returns = A.gae(seg.rewards, seg.values, seg.terminated, seg.truncated,
                                        seg.bootstrap_value, 0.99, 0.95,
                                        truncation_values=seg.truncation_values)
    st = A.ppo_update(seg, params, A.AcOpt.for_params(params, 1e-3), A.PpoConfig(),
                      O.philox_stream(1, "update"))
    for ref_net, got, init in ((a_ref, params.actor, actor), (c_ref, params.critic, critic)):
        d_ref = ref_net.flat().astype(np.float64) - init.flat()
        d_gpu = got.flat().astype(np.float64) - init.flat()
        rel = np.linalg.norm(d_gpu - d_ref) / np.linalg.norm(d_ref)
        cos = float(d_gpu @ d_ref / (np.linalg.norm(d_gpu) * np.linalg.norm(d_ref)))
        assert rel <= 0.05 and cos >= 0.999, (rel, cos)
    for k in ("policy_loss", "value_loss", "kl"):
        assert abs(getattr(st, k) - ost[k]) <= 1e-4 * max(1.0, abs(ost[k])), k


def test_sac_trajectory_x3_matches_reference(golden):
    """The reference's four-update sac_update golden trajectory on the 3xTF32
    back end (same bounds as the SIMT fp32 path)."""
    from oracle.port import philox_stream

    g = golden("sac")
    cfg = A.SacConfig(policy_frequency=2, batch_size=16)
    od, ad = 5, 2
    st = A.SacState.create(TN.ModelParams.from_numpy(TN.Arch(od, (16, 16), ad), g["actor0"]),
                           TN.ModelParams.from_numpy(TN.Arch(od + ad, (16, 16), 1), g["q10"]),
                           TN.ModelParams.from_numpy(TN.Arch(od + ad, (16, 16), 1), g["q20"]),
                           cfg)
    rng = philox_stream(1, "learner")
    for s in range(4):
        batch = {k: g[f"b{s}_{k}"] for k in ("obs", "action", "reward", "next_obs",
                                             "terminated", "n_used")}
        A.sac_update(batch, st, cfg, rng)
        np.testing.assert_allclose(st.params.q1.flat(), g[f"q1{s + 1}"], atol=2e-5)
        np.testing.assert_allclose(st.params.actor.flat(), g[f"actor{s + 1}"], atol=2e-5)
