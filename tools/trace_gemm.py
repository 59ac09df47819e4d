"""CTA-0 timeline of one tcgen05 GEMM launch per cfg2 shape (UL_TC_TRACE=1):
setup, per-k-tile TMA issue / MMA start, per-tile accumulator-ready and
epilogue-done times in microseconds from kernel entry.  Diagnostics only."""
from __future__ import annotations

import os
import sys
from pathlib import Path

os.environ.setdefault("UL_TC_TRACE", "1")
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import ctypes as C  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_30313_b200 import _dev, _lib  # noqa: E402

DT = int(os.environ.get("BENCH_DT", "1"))
EL = torch.bfloat16 if DT else torch.float32


def _lda(c):
    return (c + 7) // 8 * 8 if DT else (c + 3) // 4 * 4


def trace():
    buf = (C.c_ulonglong * 160)()
    _lib.call("ul_tc_trace", C.cast(buf, C.c_void_p))
    t = np.array(buf[:], dtype=np.float64)  # (160 slots)
    t0 = t[0]
    rel = lambda a: [round((x - t0) / 1e3, 2) if x else None for x in a]  # noqa: E731
    n = max(t[133], 1.0)
    waits = dict(ctas=int(t[133]), cta_kcycles=round(t[132] / n / 1e3, 2),
                 producer_wait=round(t[128] / t[132], 3) if t[132] else None,
                 mma_wait_full=round(t[129] / t[132], 3) if t[132] else None,
                 mma_wait_acc=round(t[130] / t[132], 3) if t[132] else None,
                 epi_wait_acc=round(t[131] / t[132], 3) if t[132] else None,
                 mma_issue=round(t[134] / t[132], 3) if t[132] else None)
    return dict(waits=waits, setup=rel([t[1]])[0], issue=rel(t[2:34]), mma=rel(t[34:66]),
                acc=rel(t[66:82]), epi=rel(t[82:98]), exit=rel([t[98]])[0],
                chunks=[rel(t[100 + 6 * c:105 + 6 * c]) for c in range(4)])


def run(name, fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    _lib.call("ul_tc_trace_reset")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    tr = trace()
    strip = lambda a: [x for x in a if x is not None]  # noqa: E731
    print(f"{name}: event {e0.elapsed_time(e1) * 1e3:.1f} us | setup {tr['setup']} | exit {tr['exit']}")
    print("  wait fractions of CTA cycles:", tr["waits"])
    print("  issue", strip(tr["issue"]))
    print("  mma  ", strip(tr["mma"]))
    print("  acc  ", strip(tr["acc"]))
    print("  epi  ", strip(tr["epi"]))
    for c, ch in enumerate(tr["chunks"]):
        print(f"  chunk{c} [start, tmem, math, staged, stored]", ch)


def main():
    rows, dev, P = 24576, "cuda", _dev.ptr
    x = torch.randn(rows, _lda(236), device=dev).to(EL)
    w = (torch.randn(512, _lda(236), device=dev) * 0.05).to(EL)
    b = torch.randn(512, device=dev)
    h = torch.empty(rows, _lda(512), device=dev, dtype=EL)
    run("fwd0", lambda: _lib.call("ul_gemm_tc", 3, 2, rows, 512, 236, P(x), x.stride(0), P(w),
                                  w.stride(0), P(h), h.stride(0), P(b), None, 0, 1, DT,
                                  _dev.stream()))
    h2 = torch.empty(rows, _lda(128), device=dev, dtype=EL)
    x2 = torch.randn(rows, _lda(257), device=dev).to(EL)
    w2 = (torch.randn(128, _lda(257), device=dev) * 0.05).to(EL)
    run("fwd2", lambda: _lib.call("ul_gemm_tc", 3, 2, rows, 128, 257, P(x2), x2.stride(0), P(w2),
                                  w2.stride(0), P(h2), h2.stride(0), P(b), None, 0, 1, DT,
                                  _dev.stream()))
    # dx2: dh1 [rows, 256] = dZ2 [rows, 128] W2 [128, 256] * elu'(h1) (BRES, K = 128)
    dz2 = torch.randn(rows, _lda(128), device=dev).to(EL)
    w2 = (torch.randn(128, _lda(256), device=dev) * 0.05).to(EL)
    h1 = torch.randn(rows, _lda(256), device=dev).to(EL)
    dx2 = torch.empty(rows, _lda(256), device=dev, dtype=EL)
    run("dx2", lambda: _lib.call("ul_gemm_tc", 1, 3, rows, 256, 128, P(dz2), dz2.stride(0), P(w2),
                                 w2.stride(0), P(dx2), dx2.stride(0), None, P(h1), h1.stride(0), 1,
                                 DT, _dev.stream()))
    dh = torch.randn(rows, _lda(512), device=dev).to(EL)
    wt = (torch.randn(512, _lda(256), device=dev) * 0.05).to(EL)
    dh1 = torch.randn(rows, _lda(256), device=dev).to(EL)
    dx = torch.empty(rows, _lda(512), device=dev, dtype=EL)
    run("dx1", lambda: _lib.call("ul_gemm_tc", 1, 3, rows, 512, 256, P(dh1), dh1.stride(0), P(wt),
                                 wt.stride(0), P(dx), dx.stride(0), None, P(h), h.stride(0), 1,
                                 DT, _dev.stream()))
    C_ = torch.empty(40, 512, 236, device=dev)
    run("dw0", lambda: _lib.call("ul_gemm_tc", 0, 0, 512, 236, rows, P(dh), dh.stride(0), P(x),
                                 x.stride(0), P(C_), 236, None, None, 0, 37, DT, _dev.stream()))


if __name__ == "__main__":
    main()
