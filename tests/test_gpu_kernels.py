"""GPU parity of the memory-bound kernels (K1-K6, K12, K13) and the fp32 MLP
(K7/K8) against the oracle and the reference golden vectors."""

import numpy as np
import pytest

from oracle import port as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2605_30313_b200 import _dev, _lib  # noqa: E402
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
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.abs(b)))) if a.size else 0.0


# ------------------------------------------------------------------- K1 / K2
def test_gae_vtrace_match_reference_goldens(golden):
    g = golden("scans")
    for i in range(int(g["n_cases"])):
        c = lambda k: g[f"c{i}_{k}"]
        tv = c("tv") if bool(c("use_tv")) else None
        adv, ret = A.gae(c("r"), c("v"), c("term"), c("trunc"), c("boot"), float(c("gamma")),
                         float(c("lam")), truncation_values=tv)
        assert rel_err(adv.cpu(), c("adv")) < 1e-5
        assert rel_err(ret.cpu(), c("ret")) < 1e-5
        vs, pg = A.vtrace(c("bl"), c("tl"), c("r"), c("v"), c("term"), c("boot"),
                          float(c("gamma")), float(c("rho")), float(c("c")),
                          truncated=c("trunc") if bool(c("vt_trunc")) else None,
                          truncation_values=tv)
        assert rel_err(vs.cpu(), c("vs")) < 1e-5
        assert rel_err(pg.cpu(), c("pg")) < 1e-5


@pytest.mark.parametrize("T,N", [(24, 4096), (1, 5), (3, 1), (64, 33), (24, 16384)])
def test_gae_vtrace_vs_oracle_shapes(T, N):
    rng = np.random.default_rng(T * 1000 + N)
    r = 0.1 * rng.normal(size=(T, N))
    v = rng.normal(size=(T, N))
    term = rng.random((T, N)) < 0.05
    trunc = (rng.random((T, N)) < 0.03) & ~term
    boot = rng.normal(size=N)
    tv = rng.normal(size=(T, N)) * trunc
    r32, v32, b32, tv32 = (x.astype(np.float32) for x in (r, v, boot, tv))
    adv, ret = A.gae(r32, v32, term, trunc, b32, 0.99, 0.95, truncation_values=tv32)
    oa, orr = O.gae(r32, v32, term, trunc, b32, 0.99, 0.95, truncation_values=tv32)
    assert rel_err(adv.cpu(), oa) < 1e-5 and rel_err(ret.cpu(), orr) < 1e-5
    bl = rng.normal(size=(T, N)).astype(np.float32)
    tl = (bl + 0.3 * rng.normal(size=(T, N))).astype(np.float32)
    vs, pg = A.vtrace(bl, tl, r32, v32, term, b32, 0.99, 1.0, 1.0, truncated=trunc,
                      truncation_values=tv32)
    ovs, opg = O.vtrace(bl, tl, r32, v32, term, b32, 0.99, 1.0, 1.0, truncated=trunc,
                        truncation_values=tv32)
    assert rel_err(vs.cpu(), ovs) < 1e-5 and rel_err(pg.cpu(), opg) < 1e-5


def test_gae_known_answer_and_errors():
    adv, ret = A.gae(np.array([[1.0]]), np.array([[0.0]]), np.zeros((1, 1), bool),
                     np.zeros((1, 1), bool), np.array([1.0]), 0.99, 0.0)
    assert float(adv.cpu()[0, 0]) == pytest.approx(1.99, rel=1e-6)
    with pytest.raises(ValueError):
        A.gae(np.zeros((3, 2)), np.zeros((4, 2)), np.zeros((3, 2), bool),
              np.zeros((3, 2), bool), np.zeros(2), 0.99, 0.95)


# --------------------------------------------------------------------- MLP
def test_mlp_forward_backward_match_reference_goldens(golden):
    g = golden("mlp")
    for i in range(int(g["n_cases"])):
        c = lambda k: g[f"c{i}_{k}"]
        dims = tuple(int(d) for d in c("dims"))
        arch = TN.Arch(dims[0], dims[1:-1], dims[-1])
        p = TN.ModelParams.from_numpy(arch, c("params"))
        y, cache = TN.forward(p, c("x").astype(np.float32))
        tol = 1e-5 if not bool(c("f64")) else 1e-5
        assert rel_err(y.cpu(), c("y")) < tol
        dx, gr = TN.backward(p, cache, c("dout"))
        assert rel_err(dx.cpu(), c("dx")) < tol
        assert rel_err(gr.flat(), c("grads")) < tol


@pytest.mark.parametrize("M,dims", [(24576, (235, 512, 256, 128, 12)), (300, (48, 256, 128, 1)),
                                    (7, (3, 5, 2))])
def test_mlp_vs_oracle_f64(M, dims):
    rng = np.random.default_rng(M)
    net = O.net_init(dims, 3)
    x = rng.normal(size=(M, dims[0])).astype(np.float32)
    dout = (rng.normal(size=(M, dims[-1])) / M).astype(np.float32)
    net64 = net.load_flat(net.flat().astype(np.float64))
    net64 = O.Net(net64.dims, [[w.astype(np.float64), b.astype(np.float64)] for w, b in net64.layers],
                  net64.log_std.astype(np.float64))
    y64, acts = O.mlp_forward(net64, x.astype(np.float64))
    dx64, g64 = O.mlp_backward(net64, x.astype(np.float64), acts, dout.astype(np.float64))
    arch = TN.Arch(dims[0], dims[1:-1], dims[-1])
    p = TN.ModelParams.from_numpy(arch, net.flat())
    y, cache = TN.forward(p, x)
    dx, gr = TN.backward(p, cache, dout)
    assert rel_err(y.cpu(), y64) < 1e-5
    assert rel_err(dx.cpu(), dx64) < 1e-5
    assert rel_err(gr.flat(), g64.flat()) < 1e-5


# ---------------------------------------------------------- K13 Adam / clip
def test_adam_bit_exact_vs_reference_goldens(golden):
    g = golden("adam")
    arch = TN.Arch(6, (8,), 3)
    p = TN.ModelParams.from_numpy(arch, g["params0"])
    opt = TN.OptState.for_params(p, 1e-3)
    for s in range(4):
        gr = TN.Grads(torch.empty_like(p.buf), arch)
        _dev.h2d(gr.buf, g[f"g{s}"].astype(np.float32))
        if s % 2:
            n = TN.clip_global_norm([gr], 1.0)
            assert n == pytest.approx(float(g[f"norm{s}"]), rel=1e-6)
        np.testing.assert_allclose(gr.flat(), g[f"gclipped{s}"], rtol=2e-7, atol=0)
        TN.adam_step(p, gr, opt, max_grad_norm=0.5 if s == 3 else 0.0)
        if s in (0, 2):  # unclipped steps: identical f32 op sequence -> bitwise
            np.testing.assert_array_equal(p.flat(), g[f"params{s + 1}"])
        else:
            np.testing.assert_allclose(p.flat(), g[f"params{s + 1}"], rtol=0, atol=1e-7)
        assert opt.t == s + 1


def test_adam_divergence_leaves_state():
    arch = TN.Arch(3, (), 2)
    p = TN.init_params(arch, 0)
    opt = TN.OptState.for_params(p, 1e-3)
    gr = TN.Grads(torch.ones_like(p.buf), arch)
    gr.buf[1] = float("nan")
    before = p.flat().copy()
    with pytest.raises(TN.DivergenceError):
        TN.adam_step(p, gr, opt)
    np.testing.assert_array_equal(p.flat(), before)
    assert opt.t == 0


def test_polyak_bitwise():
    rng = np.random.default_rng(0)
    t = rng.normal(size=1001).astype(np.float32)
    o = rng.normal(size=1001).astype(np.float32)
    td, od = torch.tensor(t, device="cuda"), torch.tensor(o, device="cuda")
    _lib.call("ul_polyak", _dev.ptr(td), _dev.ptr(od), 1001, 0.125, _dev.stream())
    ref = t.copy()
    ref *= 1.0 - 0.125
    ref += 0.125 * o
    np.testing.assert_array_equal(td.cpu().numpy(), ref)


# ------------------------------------------------------ K4/K5/K6 data path
def test_gather_rows_bit_exact():
    rng = np.random.default_rng(1)
    src = rng.normal(size=(1000, 236)).astype(np.float32)
    idx = rng.permutation(1000)[:333].astype(np.int64)
    sd = torch.tensor(src, device="cuda")
    dd = torch.zeros((333, 236), device="cuda")
    idd = torch.tensor(idx, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.call("ul_gather_rows", 1, _lib.ptr_array([_dev.ptr(sd)]), _lib.ptr_array([_dev.ptr(dd)]),
              _lib.i64_array([944]), _lib.i64_array([944]), _lib.i64_array([944]), None, _dev.ptr(idd),
              333, 0, 0, 1000, _dev.ptr(err), _dev.stream())
    np.testing.assert_array_equal(dd.cpu().numpy(), src[idx])
    assert int(err.item()) == 0


def test_device_permutation_is_permutation():
    for n in (1, 2, 17, 98304):
        out = torch.empty(n, dtype=torch.int64, device="cuda")
        _lib.call("ul_device_permutation", n, 12345, _dev.ptr(out), _dev.stream())
        np.testing.assert_array_equal(np.sort(out.cpu().numpy()), np.arange(n))


def test_normalizer_matches_reference_goldens(golden):
    g = golden("norm_replay")
    norm = TN.Normalizer(7)
    for s in range(5):
        x = g[f"n_x{s}"]
        if len(x):
            norm.update(x)
        assert norm.count == float(g[f"n_count{s}"])
        np.testing.assert_allclose(norm.mean, g[f"n_mean{s}"], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(norm.var, g[f"n_var{s}"], rtol=1e-9, atol=1e-12)
        if len(x):
            np.testing.assert_allclose(norm.apply(x).cpu().numpy(), g[f"n_apply{s}"], rtol=0,
                                       atol=2e-6)


@pytest.mark.parametrize("D", [96, 8, 200, 1100])
def test_normalizer_vectorized_moments(D):
    """K3 vectorised path (D % 4 == 0: float4 lanes, one 1024-thread CTA per SM,
    multi-phase last-CTA merge): running statistics over batches of very
    different sizes, offset far from zero (the shifted sums must not cancel),
    equal the float64 statistics of all rows seen (R:tensornet/normalizer.py:27-45)."""
    rng = np.random.default_rng(D)
    norm = TN.Normalizer(D)
    seen = []
    for B in (5000, 1, 3, 70000, 257):
        x = (100.0 + 3.0 * rng.normal(size=(B, D))).astype(np.float32)
        norm.update(x)
        seen.append(x.astype(np.float64))
        allx = np.concatenate(seen)
        assert norm.count == float(len(allx))
        np.testing.assert_allclose(norm.mean, allx.mean(0), rtol=1e-11, atol=1e-9)
        np.testing.assert_allclose(norm.var, allx.var(0), rtol=1e-7, atol=1e-9)


def test_gather_rows_cfg2_minibatch_bit_exact():
    """K4 at the cfg2 shape (98,304-row segment, one 24,576-row minibatch of a
    reference-style permutation): obs rows (944 B, with the ones column), action
    rows (48 B) and a per-row scalar gathered in one launch, bit-exact
    (gathered minibatch contents bit-exact)."""
    rng = np.random.default_rng(7)
    rows, mb = 98304, 24576
    obs = rng.normal(size=(rows, 236)).astype(np.float32)
    act = rng.normal(size=(rows, 12)).astype(np.float32)
    sc = rng.normal(size=rows).astype(np.float32)
    idx = rng.permutation(rows)[:mb].astype(np.int64)
    so, sa, ss = (torch.tensor(a, device="cuda") for a in (obs, act, sc))
    do = torch.zeros((mb, 236), device="cuda")
    da = torch.zeros((mb, 12), device="cuda")
    ds = torch.zeros(mb, device="cuda")
    idd = torch.tensor(idx, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    P = _dev.ptr
    _lib.call("ul_gather_rows", 3, _lib.ptr_array([P(so), P(sa), P(ss)]),
              _lib.ptr_array([P(do), P(da), P(ds)]), _lib.i64_array([944, 48, 4]),
              _lib.i64_array([944, 48, 4]), _lib.i64_array([944, 48, 4]),
              _lib.i64_array([4 * 235, -1, -1]), P(idd), mb, 0, 0, rows, P(err), _dev.stream())
    want = obs[idx].copy()
    want[:, 235] = 1.0
    np.testing.assert_array_equal(do.cpu().numpy(), want)
    np.testing.assert_array_equal(da.cpu().numpy(), act[idx])
    np.testing.assert_array_equal(ds.cpu().numpy(), sc[idx])
    assert int(err.item()) == 0


@pytest.mark.parametrize("cap", [1 << 20, 1000003])
def test_gather_rows_replay_ring_window(cap):
    """K6 replay sampling (R:replaypath/storage.py:106-133): absolute indices
    mapped to ring slots by idx % capacity (power-of-two capacities take the
    mask path), rows outside the [lo, hi) window skipped with the IndexError
    flag raised; in-window rows bit-exact."""
    rng = np.random.default_rng(cap % 97)
    width = 220  # RowCodec(96, 23) = 218 floats, 16-byte pitch
    ring = torch.randn(cap, width, device="cuda")
    lo, hi = 3 * cap + 11, 4 * cap + 5  # the live window after wrapping
    n = 8192
    idx = rng.integers(lo, hi, n).astype(np.int64)
    out = torch.zeros(n, width, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    P = _dev.ptr
    rb = width * 4
    args = lambda ix: (1, _lib.ptr_array([P(ring)]), _lib.ptr_array([P(out)]), _lib.i64_array([rb]),  # noqa: E731
                       _lib.i64_array([rb]), _lib.i64_array([rb]), None, P(ix), n, cap, lo, hi,
                       P(err), _dev.stream())
    _lib.call("ul_gather_rows", *args(torch.tensor(idx, device="cuda")))
    assert int(err.item()) == 0
    np.testing.assert_array_equal(out.cpu().numpy(), ring.cpu().numpy()[idx % cap])
    bad = idx.copy()
    bad[17] = hi  # one row just past the window
    out.zero_()
    _lib.call("ul_gather_rows", *args(torch.tensor(bad, device="cuda")))
    assert int(err.item()) == 1
    got = out.cpu().numpy()
    assert not got[17].any()
    keep = np.arange(n) != 17
    np.testing.assert_array_equal(got[keep], ring.cpu().numpy()[idx[keep] % cap])


@pytest.mark.parametrize("pinned", [True, False])
def test_ring_insert_matches_oracle_ring(pinned):
    """K5 device ring insert (R:replaypath/storage.py:76-104) against the
    oracle Ring over a sequence of chunks: in-place, wrapping, and a chunk
    larger than the capacity (only its tail survives, each row at its own
    absolute slot).  Source rows in pinned host memory (H2D) or HBM (D2D).
    Bit-exact."""
    from oracle.port import Ring

    cap, width = 1000, 218
    rng = np.random.default_rng(7)
    ring = torch.zeros(cap, width, device="cuda")
    ref = Ring(cap, width)
    for n in (300, 600, 250, 2345, 0, 999, 1):
        rows = rng.normal(size=(n, width)).astype(np.float32)
        if pinned:
            src = _dev.pinned_empty((max(n, 1), width), np.float32)[:n]
            src[...] = rows
            ptr = src.ctypes.data
        else:
            src = torch.from_numpy(rows).cuda() if n else torch.zeros(1, width, device="cuda")
            ptr = _dev.ptr(src)
        _lib.call("ul_ring_insert", _dev.ptr(ring), cap, width, ref.head, ptr, n, _dev.stream())
        ref.insert(rows)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(ring.cpu().numpy(), ref.data)
