"""Minibatch gather (K4) probe: cfg2 shape, sequential vs permuted indices,
fp32 rows vs 2 arrays.  CUDA-graph timed.  Diagnostics only."""
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
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record()
        g.replay()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / reps)
    return best


rows, mb, ld = 98304, 24576, 236
src = [torch.randn(rows, ld, device="cuda") for _ in range(2)]
dst = [torch.empty(mb, ld, device="cuda") for _ in range(2)]
P = _dev.ptr
for name, idx in (("seq", torch.arange(mb, device="cuda")),
                  ("perm", torch.randperm(rows, device="cuda")[:mb].contiguous())):
    for nd in (1, 2):
        f = lambda: _lib.call("ul_gather_rows", nd, _lib.ptr_array([P(t) for t in src[:nd]]),
                              _lib.ptr_array([P(t) for t in dst[:nd]]),
                              _lib.i64_array([ld * 4] * nd), _lib.i64_array([ld * 4] * nd),
                              _lib.i64_array([ld * 4] * nd), None, P(idx), mb, 0, 0, rows,
                              None, _dev.stream())
        us = timed(f)
        b = 2 * nd * mb * ld * 4
        print(f"{name} arrays={nd}: {us:.1f} us  {b / us / 1e3:.0f} GB/s")
