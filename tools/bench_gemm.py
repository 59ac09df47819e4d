"""Times the tcgen05 GEMM on the cfg2 MLP shapes (24576-row minibatch,
235-512-256-128 trunk): forward (bias+ELU), dX (ELU-grad epilogue) and dW
(split-K).  CUDA events, best of N.  The cluster size is fixed per process by
UL_TC_CLUSTER (1, 2, 4), so run once per setting.  Prints one JSON object.
"""
from __future__ import annotations

import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2605_30313_b200 import _dev, _lib  # noqa: E402


def _time(fn, reps=20, warm=3):
    """Per-launch device time: `reps` launches captured in one CUDA graph (the
    way the learner plan runs them), so host launch cost is not measured."""
    if os.environ.get("BENCH_GEMM_ONCE"):  # under ncu: one launch per shape
        fn()
        torch.cuda.synchronize()
        return 1e-9
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    best = 1e30
    s = torch.cuda.current_stream()
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        g.replay()
        e1.record(s)
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3 / reps)
    return best


DT = int(os.environ.get("BENCH_DT", "0"))  # 0: fp32 / tf32, 1: bf16
EL = torch.bfloat16 if DT else torch.float32
EB = 2 if DT else 4


def _ld(c):
    return (c + 3) // 4 * 4


def _lda(c):  # operand / activation rows: 16 bytes
    return (c + 7) // 8 * 8 if DT else (c + 3) // 4 * 4


def main():
    rows = 24576
    dims = [235, 512, 256, 128]
    dev = "cuda"
    P = _dev.ptr
    out = {"cluster_cap": os.environ.get("UL_TC_CLUSTER", "default"), "dtype": DT}
    for i in range(3):
        k, n = dims[i], dims[i + 1]
        kk = k + 1  # ones column
        x = torch.randn(rows, _lda(kk), device=dev).to(EL)
        w = (torch.randn(n, _lda(kk), device=dev) * 0.05).to(EL)
        b = torch.randn(n, device=dev)
        h = torch.empty(rows, _lda(n), device=dev, dtype=EL)
        t = _time(lambda: _lib.call("ul_gemm_tc", 3, 2, rows, n, kk, P(x), x.stride(0), P(w),
                                    w.stride(0), P(h), h.stride(0), P(b), None, 0, 1, DT, _dev.stream()))
        fl = 2.0 * rows * n * kk
        by = EB * rows * (kk + n)
        out[f"fwd{i}"] = dict(MNK=[rows, n, kk], us=t * 1e6, tflops=fl / t / 1e12,
                              gbs=by / t / 1e9)
        # dW = dH^T X : M = n (out), N = kk (in + ones), K = rows
        dh = torch.randn(rows, _lda(n), device=dev).to(EL)
        mt = -(-n // 128)
        nt = -(-kk // (256 if kk > 128 else 128))
        splits = max(1, -(-148 // (mt * nt)))
        bk = 64 if DT else 32
        kps = -(-(-(-rows // splits)) // bk) * bk
        zs = -(-rows // kps)
        C = torch.empty(zs, n, _ld(kk), device=dev)
        t = _time(lambda: _lib.call("ul_gemm_tc", 0, 0, n, kk, rows, P(dh), dh.stride(0), P(x),
                                    x.stride(0), P(C), _ld(kk), None, None, 0, splits, DT,
                                    _dev.stream()))
        fl = 2.0 * rows * n * kk
        by = EB * rows * (kk + n) + 4.0 * zs * n * kk
        out[f"dw{i}"] = dict(MNK=[n, kk, rows], splits=zs, us=t * 1e6, tflops=fl / t / 1e12,
                             gbs=by / t / 1e9)
        if i > 0:
            # dX = dH W (ELU-grad epilogue): M = rows, N = k, K = n
            wt = (torch.randn(n, _lda(k), device=dev) * 0.05).to(EL)
            hp = torch.randn(rows, _lda(k), device=dev).to(EL)
            dx = torch.empty(rows, _lda(k), device=dev, dtype=EL)
            t = _time(lambda: _lib.call("ul_gemm_tc", 1, 3, rows, k, n, P(dh), dh.stride(0),
                                        P(wt), wt.stride(0), P(dx), dx.stride(0), None, P(hp),
                                        hp.stride(0), 1, DT, _dev.stream()))
            fl = 2.0 * rows * n * k
            by = EB * rows * (n + 2 * k)
            out[f"dx{i}"] = dict(MNK=[rows, k, n], us=t * 1e6, tflops=fl / t / 1e12,
                                 gbs=by / t / 1e9)
    out["total_us"] = sum(v["us"] for v in out.values() if isinstance(v, dict))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
