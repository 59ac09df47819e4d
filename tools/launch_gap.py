"""Per-launch cost of dependent tiny kernels replayed from a CUDA graph (the
floor every extra kernel in the learner plan pays).  Diagnostics only."""
import torch

x = torch.zeros(1, device="cuda")
for n in (1, 10, 100):
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        x.add_(1)
        with torch.cuda.graph(g, stream=s):
            for _ in range(n):
                x.add_(1)
    torch.cuda.synchronize()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(20):
        e0.record()
        g.replay()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3)
    print(f"{n:4d} kernels: {best:8.2f} us total, {best / n:6.2f} us per kernel")
