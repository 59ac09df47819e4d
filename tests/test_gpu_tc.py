"""tcgen05 tensor-core GEMM (kind::tf32) parity against float64 numpy, and the
tf32 MLP / PPO paths against the oracle at the tolerance of a reduced-precision
GEMM path (north_star: 1e-2; tf32 lands near 1e-3)."""

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

TF32_TOL = 1e-2  # relative-to-max(1,|ref|) bound of the reduced-precision GEMM path


@pytest.fixture(autouse=True)
def tf32_mode():
    old = P.get_precision()
    P.set_precision("tf32")
    yield
    P.set_precision(old)


def _dev_mat(a, ld=None):
    a = np.ascontiguousarray(a, np.float32)
    r, c = a.shape
    ld = ld or ((c + 3) // 4 * 4)
    t = torch.zeros((r, ld), dtype=torch.float32, device="cuda")
    t[:, :c] = torch.from_numpy(a).cuda()
    return t


def _rel(got, ref):
    scale = max(1.0, float(np.max(np.abs(ref))))
    return float(np.max(np.abs(got - ref))) / scale


@pytest.mark.parametrize("M,N,K", [(128, 64, 32), (300, 200, 100), (24576, 512, 235),
                                   (1024, 256, 512), (4096, 128, 256)])
@pytest.mark.parametrize("epi", [0, 1, 2])
def test_tc_forward_layout(M, N, K, epi):
    """A K-major [M,K], B K-major [N,K] (the MLP forward), bias / ELU epilogues."""
    rng = np.random.default_rng(M + N + K + epi)
    a = rng.normal(size=(M, K)).astype(np.float32)
    b = (rng.normal(size=(N, K)) / np.sqrt(K)).astype(np.float32)
    bias = rng.normal(size=N).astype(np.float32)
    ref = a.astype(np.float64) @ b.astype(np.float64).T
    if epi >= 1:
        ref = ref + bias
    if epi == 2:
        ref = np.where(ref > 0, ref, np.expm1(np.minimum(ref, 0)))
    A_, B_ = _dev_mat(a), _dev_mat(b)
    C = torch.zeros((M, (N + 3) // 4 * 4), dtype=torch.float32, device="cuda")
    bd = torch.from_numpy(bias).cuda()
    _lib.call("ul_gemm_tc", 3, epi, M, N, K, _dev.ptr(A_), A_.stride(0), _dev.ptr(B_),
              B_.stride(0), _dev.ptr(C), C.stride(0), _dev.ptr(bd), None, 0, 1, 0, _dev.stream())
    got = C[:, :N].cpu().numpy()
    assert _rel(got, ref) < 2e-3


@pytest.mark.parametrize("M,N,K", [(256, 512, 256), (24576, 256, 512), (500, 96, 64)])
def test_tc_dx_layout_elu_grad(M, N, K):
    """A K-major [M,K], B N-major [K,N] (dX = dH W), ELU-gradient epilogue."""
    rng = np.random.default_rng(M * 7 + N)
    dh = rng.normal(size=(M, K)).astype(np.float32)
    w = (rng.normal(size=(K, N)) / np.sqrt(K)).astype(np.float32)
    h = np.where(rng.random((M, N)) < 0.5, rng.uniform(-0.9, 0, (M, N)),
                 rng.uniform(0, 2, (M, N))).astype(np.float32)
    ref = (dh.astype(np.float64) @ w.astype(np.float64)) * (np.minimum(h, 0) + 1.0)
    A_, B_, H_ = _dev_mat(dh), _dev_mat(w), _dev_mat(h)
    C = torch.zeros((M, (N + 3) // 4 * 4), dtype=torch.float32, device="cuda")
    _lib.call("ul_gemm_tc", 1, 3, M, N, K, _dev.ptr(A_), A_.stride(0), _dev.ptr(B_), B_.stride(0),
              _dev.ptr(C), C.stride(0), None, _dev.ptr(H_), H_.stride(0), 1, 0, _dev.stream())
    assert _rel(C[:, :N].cpu().numpy(), ref) < 2e-3


@pytest.mark.parametrize("out,inp,rows,splits", [(512, 236, 24576, 37), (128, 64, 1000, 1),
                                                 (256, 513, 4096, 8)])
def test_tc_dw_layout_split_k(out, inp, rows, splits):
    """A M-major (dH [rows,out] read transposed), B N-major (H [rows,in]):
    dW = dH^T H with split-K partials."""
    rng = np.random.default_rng(out + inp)
    dh = (rng.normal(size=(rows, out)) / np.sqrt(rows)).astype(np.float32)
    x = rng.normal(size=(rows, inp)).astype(np.float32)
    ref = dh.astype(np.float64).T @ x.astype(np.float64)
    A_, B_ = _dev_mat(dh), _dev_mat(x)
    kps = -(-(-(-rows // splits)) // 32) * 32  # split length, rounded to the 32-row K tile
    zs = -(-rows // kps)
    ldc = (inp + 3) // 4 * 4  # split partials: [zs][out][ldc], 16 B rows
    C = torch.zeros((zs, out, ldc), dtype=torch.float32, device="cuda")
    _lib.call("ul_gemm_tc", 0, 0, out, inp, rows, _dev.ptr(A_), A_.stride(0), _dev.ptr(B_),
              B_.stride(0), _dev.ptr(C), ldc, None, None, 0, splits, 0, _dev.stream())
    got = C.sum(0)[:, :inp].cpu().numpy()
    assert _rel(got, ref) < 2e-3


@pytest.mark.parametrize("M,dims", [(24576, (235, 512, 256, 128, 12)), (512, (48, 256, 128, 1))])
def test_mlp_tf32_vs_oracle_f64(M, dims):
    rng = np.random.default_rng(M)
    net = O.net_init(dims, 3)
    x = rng.normal(size=(M, dims[0])).astype(np.float32)
    dout = (rng.normal(size=(M, dims[-1])) / M).astype(np.float32)
    net64 = O.Net(net.dims, [[w.astype(np.float64), b.astype(np.float64)] for w, b in net.layers],
                  net.log_std.astype(np.float64))
    y64, acts = O.mlp_forward(net64, x.astype(np.float64))
    dx64, g64 = O.mlp_backward(net64, x.astype(np.float64), acts, dout.astype(np.float64))
    p = TN.ModelParams.from_numpy(TN.Arch(dims[0], dims[1:-1], dims[-1]), net.flat())
    y, cache = TN.forward(p, x)
    dx, gr = TN.backward(p, cache, dout)
    assert _rel(y.cpu().numpy(), y64) < TF32_TOL
    assert _rel(dx.cpu().numpy(), dx64) < TF32_TOL
    g = gr.flat()
    for (w, b), off in zip(g64.layers, np.cumsum([0] + [w.size + b.size for w, b in g64.layers])[:-1]):
        gw = g[off:off + w.size].reshape(w.shape)
        gb = g[off + w.size:off + w.size + b.size]
        assert _rel(gw, w) < TF32_TOL
        assert _rel(gb, b) < TF32_TOL
