"""Per-launch fixed cost of the tcgen05 GEMM at cfg2 shapes: the same GEMM
replayed back to back in a CUDA graph at M = 24,576 rows (one minibatch) and
at 8x the rows; (t(M) - t(8M)/8) is the launch's fill / drain / transition
cost.  Diagnostics only."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_30313_b200 import _dev, _lib  # noqa: E402


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / reps)
    return best


def lda(c):
    return (c + 7) // 8 * 8


P = _dev.ptr
dev = "cuda"
for name, K, N, epi in (("fwd L1 512->256 bias+ELU", 512, 256, 2), ("fwd L2 256->128", 256, 128, 2),
                        ("fwd L0 235->512", 235, 512, 2)):
    res = []
    for mult in (1, 8):
        M = 24576 * mult
        x = torch.randn(M, lda(K + 1), device=dev).to(torch.bfloat16)
        w = (torch.randn(N, lda(K + 1), device=dev) * 0.05).to(torch.bfloat16)
        b = torch.randn(N, device=dev)
        h = torch.empty(M, lda(N + 1), device=dev, dtype=torch.bfloat16)
        fn = lambda: _lib.call("ul_gemm_tc", 3, epi, M, N, K, P(x), x.stride(0), P(w),  # noqa: E731
                               w.stride(0), P(h), h.stride(0), P(b), None, 0, 1, 1,
                               torch.cuda.current_stream().cuda_stream)
        res.append(timed(fn))
    t1, t8 = res
    print(f"{name}: {t1:.2f} us per 24576-row launch, {t8 / 8:.2f} us per 24576 rows at 8x "
          f"-> fixed cost {t1 - t8 / 8:.2f} us")
