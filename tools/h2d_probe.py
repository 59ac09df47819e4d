"""PCIe H2D bandwidth of one cfg2 segment's bytes (192 MB pinned -> HBM):
one copy stream vs the copy split across 2 / 4 streams, alone and while the
graphed cfg2 update loop runs on the compute stream."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_30313_b200 as PKG  # noqa: E402
from paper_2605_30313_b200 import _dev, _lib, algos as A, tensornet as TN  # noqa: E402
from paper_2605_30313_b200.algos import ppo as P  # noqa: E402
from paper_2605_30313_b200.algos._staging import staging_for  # noqa: E402
from paper_2605_30313_b200.workload import CONFIGS, make_rollout  # noqa: E402

NB = 192 << 20
host = _dev.pinned_empty((NB,), np.uint8)
host[...] = 1
dev = torch.empty(NB, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]


def copy(nstreams, chunk_mb=None):
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    s0 = streams[0]
    ev0.record(s0)
    for s in streams[1:nstreams]:
        s.wait_event(ev0)
    chunk = (chunk_mb << 20) if chunk_mb else NB // nstreams
    off, i = 0, 0
    while off < NB:
        n = min(chunk, NB - off)
        s = streams[i % nstreams]
        _lib.call("ul_memcpy_async", _dev.ptr(dev) + off, host.ctypes.data + off, n, s.cuda_stream)
        off += n
        i += 1
    for s in streams[1:nstreams]:
        ev = torch.cuda.Event()
        ev.record(s)
        s0.wait_event(ev)
    ev1.record(s0)
    return ev0, ev1


def bw(nstreams, chunk_mb=None, reps=5):
    out = []
    for _ in range(reps):
        e0, e1 = copy(nstreams, chunk_mb)
        torch.cuda.synchronize()
        out.append(NB / (e0.elapsed_time(e1) / 1e3) / 1e9)
    return max(out)


for ns, ch in ((1, None), (2, None), (4, None), (1, 8), (2, 8), (4, 8)):
    print(f"alone  streams={ns} chunk={ch or 'split'}MB: {bw(ns, ch):.1f} GB/s")

PKG.set_precision("bf16")
T, N, od, cd, ad, hid = CONFIGS["cfg2"]
cfg = A.PpoConfig()
params = A.AcParams(TN.init_params(TN.Arch(od, hid, ad), 0), TN.init_params(TN.Arch(cd, hid, 1), 1))
opt = A.AcOpt.for_params(params, cfg.lr)
w = make_rollout("cfg2", 0)
seg = A.RolloutSegment(obs=w.obs, critic_obs=w.critic_obs, actions=w.actions,
                       behavior_log_prob=np.zeros((T, N)) - 15.0, rewards=w.rewards,
                       terminated=w.terminated, truncated=w.truncated, values=np.zeros((T, N)),
                       bootstrap_value=w.bootstrap_value, truncation_values=w.truncation_values)
ds = staging_for(T, N, od, cd, ad, cfg.epochs)
ds.load(seg, with_advantages=False)
rng = A.DeviceRng(1)
for _ in range(3):
    P.ppo_update_resident(ds, params, opt, cfg, rng)
torch.cuda.synchronize()
for ns, ch in ((1, None), (2, None), (4, None), (2, 8)):
    res = []
    for _ in range(3):
        for _ in range(3):  # ~14 ms of updates queued ahead of the copy
            P.ppo_update_resident(ds, params, opt, cfg, rng)
        e0, e1 = copy(ns, ch)
        torch.cuda.synchronize()
        res.append(NB / (e0.elapsed_time(e1) / 1e3) / 1e9)
    print(f"under update  streams={ns} chunk={ch or 'split'}MB: {max(res):.1f} GB/s (min {min(res):.1f})")
