"""bf16 tensor-core path (tcgen05 kind::f16, fp32 accumulation): the GEMM
layouts/epilogues against float64 numpy on the same bf16-rounded operands, and
the bf16 PPO update against the oracle at the north-star tolerance of bf16 GEMM
paths (1e-2 on losses; parameter-delta direction within the full-update bound
of SURVEY.md 8(c), loosened for bf16 activations)."""

import numpy as np
import pytest

from oracle import port as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2605_30313_b200 as P  # noqa: E402
from paper_2605_30313_b200 import _dev, _lib  # noqa: E402
from paper_2605_30313_b200 import algos as A  # noqa: E402
from paper_2605_30313_b200 import tensornet as TN  # noqa: E402

BF16_TOL = 1e-2  # relative-to-max(1,|ref|) bound of the bf16 GEMM path (north_star)


@pytest.fixture
def bf16_mode():
    old = P.get_precision()
    P.set_precision("bf16")
    yield
    P.set_precision(old)


def _bf(a, ld=None):
    """bf16 device copy [rows, ld] (pad zero) and its exact float64 value."""
    a = np.ascontiguousarray(a, np.float32)
    r, c = a.shape
    ld = ld or ((c + 7) // 8 * 8)
    t = torch.zeros((r, ld), dtype=torch.bfloat16, device="cuda")
    t[:, :c] = torch.from_numpy(a).cuda().to(torch.bfloat16)
    return t, t[:, :c].float().cpu().numpy().astype(np.float64)


def _rel(got, ref):
    scale = max(1.0, float(np.max(np.abs(ref))))
    return float(np.max(np.abs(got - ref))) / scale


@pytest.mark.parametrize("M,N,K", [(128, 64, 32), (300, 200, 100), (24576, 512, 236),
                                   (1024, 256, 513), (77, 12, 40), (4096, 128, 257)])
@pytest.mark.parametrize("epi", [0, 1, 2])
def test_bf16_forward_layout(M, N, K, epi):
    """A K-major [M,K], B K-major [N,K]; epilogue 2 (bias+ELU) writes bf16."""
    rng = np.random.default_rng(M + N + K + epi)
    A_, a = _bf(rng.normal(size=(M, K)))
    B_, b = _bf(rng.normal(size=(N, K)) / np.sqrt(K))
    bias = rng.normal(size=N).astype(np.float32)
    ref = a @ b.T
    if epi >= 1:
        ref = ref + bias
    if epi == 2:
        ref = np.where(ref > 0, ref, np.expm1(np.minimum(ref, 0)))
    if epi == 2:
        C = torch.zeros((M, (N + 7) // 8 * 8), dtype=torch.bfloat16, device="cuda")
    else:
        C = torch.zeros((M, (N + 3) // 4 * 4), dtype=torch.float32, device="cuda")
    bd = torch.from_numpy(bias).cuda()
    _lib.call("ul_gemm_tc", 3, epi, M, N, K, _dev.ptr(A_), A_.stride(0), _dev.ptr(B_),
              B_.stride(0), _dev.ptr(C), C.stride(0), _dev.ptr(bd), None, 0, 1, 1, _dev.stream())
    got = C[:, :N].float().cpu().numpy()
    assert _rel(got, ref) < (1e-2 if epi == 2 else 2e-5 * np.sqrt(K) + 1e-5)


@pytest.mark.parametrize("M,N,K", [(256, 512, 256), (24576, 256, 512), (500, 96, 64),
                                   (24576, 128, 256)])
def test_bf16_dx_layout_elu_grad(M, N, K):
    """A K-major [M,K] (dH), B N-major [K,N] (W), ELU-gradient epilogue, bf16 in/out."""
    rng = np.random.default_rng(M * 7 + N)
    dH, dh = _bf(rng.normal(size=(M, K)))
    W, w = _bf(rng.normal(size=(K, N)) / np.sqrt(K))
    H, h = _bf(np.where(rng.random((M, N)) < 0.5, rng.uniform(-0.9, 0, (M, N)),
                        rng.uniform(0, 2, (M, N))))
    ref = (dh @ w) * (np.minimum(h, 0) + 1.0)
    C = torch.zeros((M, (N + 7) // 8 * 8), dtype=torch.bfloat16, device="cuda")
    _lib.call("ul_gemm_tc", 1, 3, M, N, K, _dev.ptr(dH), dH.stride(0), _dev.ptr(W), W.stride(0),
              _dev.ptr(C), C.stride(0), None, _dev.ptr(H), H.stride(0), 1, 1, _dev.stream())
    assert _rel(C[:, :N].float().cpu().numpy(), ref) < 1e-2


@pytest.mark.parametrize("out,inp,rows,splits", [(512, 236, 24576, 37), (128, 64, 1000, 1),
                                                 (256, 513, 4096, 8), (12, 49, 600, 3)])
def test_bf16_dw_layout_split_k(out, inp, rows, splits):
    """A M-major (dH [rows,out] read transposed), B N-major (H [rows,in]):
    dW = dH^T H with split-K fp32 partials."""
    rng = np.random.default_rng(out + inp)
    dH, dh = _bf(rng.normal(size=(rows, out)) / np.sqrt(rows))
    X, x = _bf(rng.normal(size=(rows, inp)))
    ref = dh.T @ x
    kps = -(-(-(-rows // splits)) // 64) * 64  # split length, rounded to the 64-row bf16 K tile
    zs = -(-rows // kps)
    ldc = (inp + 3) // 4 * 4
    C = torch.zeros((zs, out, ldc), dtype=torch.float32, device="cuda")
    _lib.call("ul_gemm_tc", 0, 0, out, inp, rows, _dev.ptr(dH), dH.stride(0), _dev.ptr(X),
              X.stride(0), _dev.ptr(C), ldc, None, None, 0, splits, 1, _dev.stream())
    got = C.sum(0)[:, :inp].cpu().numpy()
    assert _rel(got, ref) < 1e-4


def test_ppo_update_bf16_small_net(bf16_mode):
    """cfg1-shaped nets (48 -> 256-128-128): first-layer dW with N = 49 < one
    tile and db through skinny-fused column sums."""
    from oracle.port import philox_stream
    from helpers import _synthetic

    T, N = 8, 256
    segd, actor, critic = _synthetic(T, N, 48, 48, 12, (256, 128, 128), seed=4)
    adv, ret = O.gae(segd["rewards"], segd["values"], segd["terminated"], segd["truncated"],
                     segd["bootstrap_value"], 0.99, 0.95, segd["truncation_values"])
    cfg = O.PpoCfg(epochs=1, minibatches=2)
    a_ref, c_ref = actor.clone(), critic.clone()
    oa, oc = O.Opt.for_net(a_ref, cfg.lr), O.Opt.for_net(c_ref, cfg.lr)
    O.ppo_update(dict(segd, advantages=adv, returns=ret), a_ref, c_ref, oa, oc, cfg,
                 philox_stream(3, "update"))
    params = A.AcParams(TN.ModelParams.from_numpy(TN.Arch(48, (256, 128, 128), 12), actor.flat()),
                        TN.ModelParams.from_numpy(TN.Arch(48, (256, 128, 128), 1), critic.flat()))
    seg = A.RolloutSegment(**segd)
    seg.advantages, seg.returns = A.gae(seg.rewards, seg.values, seg.terminated, seg.truncated,
                                        seg.bootstrap_value, 0.99, 0.95,
                                        truncation_values=seg.truncation_values)
    opt = A.AcOpt.for_params(params, 1e-3)
    A.ppo_update(seg, params, opt, A.PpoConfig(epochs=1, minibatches=2), philox_stream(3, "update"))
    for ref_net, got, init in ((a_ref, params.actor, actor), (c_ref, params.critic, critic)):
        d_ref = ref_net.flat() - init.flat()
        d_gpu = got.flat() - init.flat()
        cos = float(d_gpu @ d_ref / (np.linalg.norm(d_gpu) * np.linalg.norm(d_ref)))
        assert cos >= 0.97, cos


def _blocks(flat, dims):
    """Split a ModelParams.flat() vector into its [W_i, b_i ..., log_std] blocks
    (R:tensornet/mlp.py:53-57 order)."""
    out, o = [], 0
    for i in range(len(dims) - 1):
        for n in (dims[i + 1] * dims[i], dims[i + 1]):
            out.append(flat[o:o + n])
            o += n
    out.append(flat[o:o + dims[-1]])
    return out


@pytest.mark.parametrize("hidden,act_dim,cobs", [((512, 256, 128), 12, None),
                                                 ((256, 128, 128), 12, None),
                                                 ((512, 256, 128), 29, 101)])
def test_ppo_single_step_grads_bf16_per_layer(bf16_mode, hidden, act_dim, cobs):
    """One minibatch's gradients on the bf16 path (fused output stage, batched
    dW, ELU-gradient dX) against the f64 oracle, block by block: every W, b and
    log_std of both networks within 3e-2 relative norm error, so an error in a
    small block (the 12 x 128 output layer) cannot hide in a whole-net norm."""
    from helpers import _synthetic

    T, N = 8, 1024
    od = 235 if hidden[0] == 512 else 48
    if act_dim == 29:  # cfg5 (G1 humanoid) shapes: obs 98 / critic obs 101 / 29 actions
        od = 98
    cd = cobs or od
    seg, actor, critic = _synthetic(T, N, od, cd, act_dim, hidden, seed=5)
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
    params = A.AcParams(TN.ModelParams.from_numpy(TN.Arch(od, hidden, act_dim), actor.flat()),
                        TN.ModelParams.from_numpy(TN.Arch(cd, hidden, 1), critic.flat()))
    gterms, gga, ggc = A.ppo_loss_and_grads(params, f(seg["obs"]), f(seg["critic_obs"]),
                                            f(seg["actions"]), seg["behavior_log_prob"].reshape(-1),
                                            advn, ret.reshape(-1), seg["values"].reshape(-1),
                                            A.PpoConfig())
    for k in ("policy_loss", "value_loss", "kl"):
        assert abs(gterms[k] - terms[k]) <= BF16_TOL * max(1.0, abs(terms[k])), k
    for ref, got, dims in ((ga, gga, (od, *hidden, act_dim)), (gc, ggc, (cd, *hidden, 1))):
        for i, (r, g) in enumerate(zip(_blocks(np.asarray(ref.flat(), np.float64), dims),
                                       _blocks(np.asarray(got.flat(), np.float64), dims))):
            nr = np.linalg.norm(r)
            if nr == 0.0:  # the critic's log_std
                assert np.all(g == 0.0)
                continue
            assert np.linalg.norm(g - r) / nr < 3e-2, (dims, i, np.linalg.norm(g - r) / nr)
