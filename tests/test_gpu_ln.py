"""LayerNorm hidden layers (cfg3's FastSAC critics; SURVEY.md 8(a) "bias+ELU/
LayerNorm"): forward and backward of an LN MLP through ul_mlp_forward /
ul_mlp_backward against a float64 composition of the oracle's linear / LN /
ELU pieces (oracle/port.py ln_forward, ln_backward -- pinned by finite
differences in tests/test_oracle_pinned.py).  fp32 SIMT and tf32 tensor cores at
tight tolerance, bf16 at the north-star 1e-2."""

import numpy as np
import pytest

from oracle import port as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2605_30313_b200 as P  # noqa: E402
from paper_2605_30313_b200 import tensornet as TN  # noqa: E402

# relative to the largest |reference| entry of each checked tensor
TOL = {"fp32": 1e-4, "tf32": 5e-3, "bf16": 3e-2}


def _ref(params, x, dout):
    """float64 forward/backward of the LN MLP: returns out, dx, flat grads."""
    arch = params.arch
    layers, log_std, lns = TN.mlp._views(params.buf.cpu().double(), arch, with_ln=True)
    layers = [(w.numpy(), b.numpy()) for w, b in layers]
    lns = [(g.numpy(), be.numpy()) for g, be in lns]
    h = np.asarray(x, np.float64)
    caches = []
    for k, (w, b) in enumerate(layers):
        a = h @ w.T + b
        if k < len(layers) - 1:
            n, c = O.ln_forward(a, lns[k][0], lns[k][1])
            hn = O.elu(n)
            caches.append((h, c, hn))
            h = hn
        else:
            caches.append((h, None, None))
            h = a
    out = h
    d = np.asarray(dout, np.float64)
    grads = [None] * len(layers)
    lngr = [None] * len(lns)
    for k in range(len(layers) - 1, -1, -1):
        hin, c, hn = caches[k]
        if k < len(layers) - 1:
            dn = d * O.elu_grad_from_act(hn)
            d, dg, dbeta = O.ln_backward(dn, lns[k][0], c)
            lngr[k] = (dg, dbeta)
        w, _ = layers[k]
        grads[k] = (d.T @ hin, d.sum(0))
        d = d @ w
    parts = []
    for k, (dw, db) in enumerate(grads):
        parts += [dw.ravel(), db]
        if k < len(lns):
            parts += [lngr[k][0], lngr[k][1]]
    parts.append(np.zeros(arch.output_dim))
    return out, d, np.concatenate(parts)


def _rel(got, ref):
    return float(np.max(np.abs(got - ref))) / (float(np.max(np.abs(ref))) + 1e-30)


@pytest.mark.parametrize("prec", ["fp32", "tf32", "bf16"])
@pytest.mark.parametrize("dims,rows", [((235, (512, 256, 128), 12), 1000),
                                       ((48, (256, 256), 1), 4096),
                                       ((20, (64,), 4), 37),
                                       ((16, (1028, 100), 3), 300),  # generic LN kernels
                                       ((119, (1024, 512, 256), 1), 2048)])  # cfg3 critic
def test_ln_mlp_matches_oracle(prec, dims, rows):
    inp, hid, outd = dims
    arch = TN.Arch(input_dim=inp, hidden_dims=hid, output_dim=outd, layer_norm=True)
    params = TN.init_params(arch, seed=rows + inp)
    rng = np.random.default_rng(7)
    # non-trivial gain / shift so both LN gradients are exercised
    with torch.no_grad():
        for g, be in params.layer_norms:
            g.copy_(torch.from_numpy(rng.uniform(0.5, 1.5, g.shape[0]).astype(np.float32)))
            be.copy_(torch.from_numpy(rng.normal(0, 0.2, be.shape[0]).astype(np.float32)))
    x = rng.normal(size=(rows, inp)).astype(np.float32)
    dout = rng.normal(size=(rows, outd)).astype(np.float32) / rows
    old = P.get_precision()
    P.set_precision(prec)
    try:
        out, cache = TN.forward(params, x)
        dx, grads = TN.backward(params, cache, dout)
        torch.cuda.synchronize()
    finally:
        P.set_precision(old)
    r_out, r_dx, r_g = _ref(params, x, dout)
    tol = TOL[prec]
    assert _rel(out.cpu().numpy(), r_out) < tol
    assert _rel(dx.cpu().numpy(), r_dx) < tol
    g = grads.buf.cpu().numpy()
    assert g.shape == r_g.shape
    # per-segment check so a wrong LN gain/shift gradient is not hidden by W's scale
    layers, _, lns = TN.mlp._views(torch.from_numpy(g), arch, with_ln=True)
    rl, _, rln = TN.mlp._views(torch.from_numpy(r_g), arch, with_ln=True)
    for (w, b), (rw, rb) in zip(layers, rl):
        assert _rel(w.numpy(), rw.numpy()) < tol
        assert _rel(b.numpy(), rb.numpy()) < tol
    for (gg, gb), (rg, rb) in zip(lns, rln):
        assert _rel(gg.numpy(), rg.numpy()) < tol
        assert _rel(gb.numpy(), rb.numpy()) < tol


def test_ln_param_layout_and_init():
    arch = TN.Arch(input_dim=10, hidden_dims=(16, 8), output_dim=3, layer_norm=True)
    assert arch.param_count == 16 * 10 + 16 + 32 + 8 * 16 + 8 + 16 + 3 * 8 + 3 + 3
    p = TN.init_params(arch, seed=0)
    (g0, b0), (g1, b1) = p.layer_norms
    assert torch.all(g0 == 1) and torch.all(b0 == 0) and g1.shape[0] == 8


@pytest.mark.parametrize("dims,rows", [((119, (1024, 512, 256), 1), 8192),
                                       ((48, (256, 256), 1), 1000),
                                       ((40, (640, 96), 2), 777)])
def test_ln_fused_epilogue_matches_separate_kernels(dims, rows, monkeypatch):
    """bf16: the whole LayerNorm forward inside the tcgen05 epilogue
    (kEpiLnFull: row statistics merged across a cluster of N-tile CTAs through
    distributed shared memory, h = elu(LN(a) g + beta) written by the GEMM)
    against the GEMM + separate row / column LN kernels (UL_LN_FUSED=0).
    Both normalise the same bf16 pre-LN rows; the statistics differ only in
    fp32 summation order, so outputs agree to a bf16 ulp, and the backward
    (which reads the stored rows and statistics) to the same level."""
    inp, hid, outd = dims
    arch = TN.Arch(input_dim=inp, hidden_dims=hid, output_dim=outd, layer_norm=True)
    params = TN.init_params(arch, seed=5)
    rng = np.random.default_rng(3)
    with torch.no_grad():
        for g, be in params.layer_norms:
            g.copy_(torch.from_numpy(rng.uniform(0.5, 1.5, g.shape[0]).astype(np.float32)))
            be.copy_(torch.from_numpy(rng.normal(0, 0.2, be.shape[0]).astype(np.float32)))
    x = rng.normal(size=(rows, inp)).astype(np.float32)
    dout = rng.normal(size=(rows, outd)).astype(np.float32) / rows
    old = P.get_precision()
    P.set_precision("bf16")
    res = {}
    try:
        for fused in ("0", "1"):
            monkeypatch.setenv("UL_LN_FUSED", fused)
            out, cache = TN.forward(params, x)
            dx, grads = TN.backward(params, cache, dout)
            torch.cuda.synchronize()
            res[fused] = (out.cpu().numpy(), dx.cpu().numpy(), grads.buf.cpu().numpy())
    finally:
        P.set_precision(old)
    for a, b in zip(res["0"], res["1"]):
        assert np.all(np.isfinite(b))
        assert _rel(b, a) < 2e-2, _rel(b, a)
