"""HBM-roofline microbenchmarks of the memory-bound learner kernels at sizes
larger than L2 (126 MB), CUDA events on the launching stream, best of N.

Algorithmic bytes: GAE 22 B/element (+4 B/env), V-trace
30 B/element, gather 2 x rows x row_bytes + 8 B/index, Welford 4 B/element,
Adam 28 B/param, Polyak 12 B/param.  Prints one JSON object.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_30313_b200 import _dev, _lib  # noqa: E402


def _time(fn, reps=10, warm=3, back_to_back=10):
    """Best of `reps` per-launch device times, each the mean of `back_to_back`
    consecutive launches between two events (so a short kernel's time is not
    the host launch latency the first event waits through)."""
    s = torch.cuda.current_stream()
    for _ in range(warm):
        fn()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(back_to_back):
            fn()
        e1.record(s)
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3 / back_to_back)
    return best


def run(peak_gbs: float) -> dict:
    dev = "cuda"
    out = {}
    st = _dev.stream()

    # K1 / K2 scans, [24, 2^22] (2.2 GB / 3.0 GB of traffic)
    T, N = 24, 1 << 22
    r = torch.randn(T, N, device=dev)
    v = torch.randn(T, N, device=dev)
    tv = torch.randn(T, N, device=dev)
    bl, tl = torch.randn(T, N, device=dev), torch.randn(T, N, device=dev)
    term = (torch.rand(T, N, device=dev) < 0.01).to(torch.uint8)
    trunc = (torch.rand(T, N, device=dev) < 0.005).to(torch.uint8)
    boot = torch.randn(N, device=dev)
    a1, a2 = torch.empty_like(r), torch.empty_like(r)
    P = _dev.ptr
    t = _time(lambda: _lib.call("ul_gae_f32", P(r), P(v), P(term), P(trunc), P(tv), P(boot), T, N,
                                0.99, 0.95, P(a1), P(a2), st))
    b = 22 * T * N + 4 * N
    out["gae"] = dict(shape=[T, N], seconds=t, gbs=b / t / 1e9, frac=b / t / 1e9 / peak_gbs)
    t = _time(lambda: _lib.call("ul_vtrace_f32", P(bl), P(tl), P(r), P(v), P(term), P(trunc),
                                P(tv), P(boot), T, N, 0.99, 1.0, 1.0, P(a1), P(a2), st))
    b = 30 * T * N + 4 * N
    out["vtrace"] = dict(shape=[T, N], seconds=t, gbs=b / t / 1e9, frac=b / t / 1e9 / peak_gbs)
    del r, v, tv, bl, tl, term, trunc, a1, a2

    # K4 minibatch gather: cfg2 segment obs + critic_obs rows (944 B), 24,576 of 98,304
    rows, ld, mb = 98304, 236, 24576
    seg = torch.randn(2, rows, ld, device=dev)
    dst = torch.empty(2, mb, ld, device=dev)
    idx = torch.from_numpy(np.random.default_rng(0).permutation(rows)[:mb]).to(dev)
    rb = ld * 4
    srcs = _lib.ptr_array([P(seg[0]), P(seg[1])])
    dsts = _lib.ptr_array([P(dst[0]), P(dst[1])])
    st_b = _lib.i64_array([rb, rb])
    t = _time(lambda: _lib.call("ul_gather_rows", 2, srcs, dsts, st_b, st_b, st_b, None, P(idx),
                                mb, 0, 0, rows, None, st))
    b = 2 * (2 * mb * rb) + 8 * mb
    out["gather_minibatch"] = dict(rows=mb, row_bytes=rb, arrays=2, seconds=t, gbs=b / t / 1e9,
                                   frac=b / t / 1e9 / peak_gbs)
    del seg, dst

    # K6 replay sample gather: 1M-row ring of 880 B rows (cfg3), 32,768 samples x 8 batches
    cap, pitch, n = 1 << 20, 220, 32768 * 8
    ring = torch.randn(cap, pitch, device=dev)
    outb = torch.empty(n, pitch, device=dev)
    ridx = torch.from_numpy(np.random.default_rng(1).integers(0, cap, n)).to(dev)
    rb = pitch * 4
    t = _time(lambda: _lib.call("ul_gather_rows", 1, _lib.ptr_array([P(ring)]),
                                _lib.ptr_array([P(outb)]), _lib.i64_array([rb]),
                                _lib.i64_array([rb]), _lib.i64_array([rb]), None, P(ridx), n, cap,
                                0, cap, None, st))
    b = 2 * n * rb + 8 * n
    out["gather_replay"] = dict(rows=n, row_bytes=rb, seconds=t, gbs=b / t / 1e9,
                                frac=b / t / 1e9 / peak_gbs)
    del ring, outb

    # K3 normaliser moments: [1M, 96] rows
    B, D = 1 << 20, 96
    x = torch.randn(B, D, device=dev)
    state = torch.zeros(1 + 2 * D, dtype=torch.float64, device=dev)
    work = torch.zeros(_lib.lib().ul_norm_work_bytes(D), dtype=torch.uint8, device=dev)
    t = _time(lambda: _lib.call("ul_norm_update", P(x), B, D, D, P(state), P(work), 0, st))
    b = 4 * B * D
    out["welford_update"] = dict(shape=[B, D], seconds=t, gbs=b / t / 1e9,
                                 frac=b / t / 1e9 / peak_gbs)
    del x

    # K12 Polyak + K13 Adam over 64M parameters
    n = 1 << 26
    p1, p2 = torch.randn(n, device=dev), torch.randn(n, device=dev)
    t = _time(lambda: _lib.call("ul_polyak", P(p1), P(p2), n, 0.01, st))
    out["polyak"] = dict(params=n, seconds=t, gbs=12 * n / t / 1e9, frac=12 * n / t / 1e9 / peak_gbs)
    g, m, vv = torch.randn(n, device=dev) * 1e-3, torch.zeros(n, device=dev), torch.zeros(n, device=dev)
    ctl = _lib.OptCtl()
    import ctypes as C

    lr = (C.c_double * 1)(1e-3)
    _lib.call("ul_opt_ctl_init", C.byref(ctl), 1, lr, 0.9, 0.999, 1e-8, 0.0)
    dctl = torch.zeros(C.sizeof(_lib.OptCtl), dtype=torch.uint8, device=dev)
    _dev.h2d(dctl, np.frombuffer(bytes(ctl), dtype=np.uint8))
    t = _time(lambda: _lib.call("ul_adam_step", _lib.ptr_array([P(p1)]), _lib.ptr_array([P(g)]),
                                _lib.ptr_array([P(m)]), _lib.ptr_array([P(vv)]),
                                _lib.i64_array([n]), 1, P(dctl), 0, st))
    b = 28 * n + 4 * n  # prepare pass reads g once more
    out["adam"] = dict(params=n, seconds=t, gbs=b / t / 1e9, frac=b / t / 1e9 / peak_gbs)
    return out


if __name__ == "__main__":
    peaks = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text())
    print(json.dumps(run(peaks["hbm_gbs"])))
