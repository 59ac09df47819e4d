"""bench.py's e2e loop (PpoPipeline.update_async from pinned host buffers, cfg2
bf16) with device events: per update the compute-stream span from the wait on
the staged segment to the end of the graph, the copy-stream span of the next
segment's staging, and the idle time between updates."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_30313_b200 as PKG  # noqa: E402
from paper_2605_30313_b200 import _dev, algos as A, tensornet as TN  # noqa: E402
from paper_2605_30313_b200.algos import ppo as P  # noqa: E402
from paper_2605_30313_b200.workload import CONFIGS, make_rollout  # noqa: E402

PKG.set_precision("bf16")
T, N, od, cd, ad, hid = CONFIGS["cfg2"]
cfg = A.PpoConfig()
params = A.AcParams(TN.init_params(TN.Arch(od, hid, ad), 0), TN.init_params(TN.Arch(cd, hid, 1), 1))
opt = A.AcOpt.for_params(params, cfg.lr)
w = make_rollout("cfg2", seed=0, alloc=_dev.pinned_empty)
w.behavior_log_prob = _dev.pinned_empty((T, N), np.float64)
w.behavior_log_prob[...] = -15.0
w.values = _dev.pinned_empty((T, N), np.float64)
w.values[...] = 0.0
seg = A.RolloutSegment(obs=w.obs, critic_obs=w.critic_obs, actions=w.actions,
                       behavior_log_prob=w.behavior_log_prob, rewards=w.rewards,
                       terminated=w.terminated, truncated=w.truncated, values=w.values,
                       bootstrap_value=w.bootstrap_value, truncation_values=w.truncation_values)
pipe = A.PpoPipeline(params, opt, cfg, A.DeviceRng(1))
for _ in range(2):
    pipe.prefetch(seg)
    pipe.update()
torch.cuda.synchronize()

marks = []  # (name, event, stream)


def ev(name, stream):
    e = torch.cuda.Event(enable_timing=True)
    e.record(stream)
    marks.append((name, e))


orig_load = None
from paper_2605_30313_b200.algos import _staging  # noqa: E402

orig_load = _staging.DeviceSegment.load if hasattr(_staging, "DeviceSegment") else None
K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
t0 = time.perf_counter()
pipe.prefetch(seg)
pend = None
for i in range(K):
    ev("async_call", torch.cuda.current_stream())
    h = pipe.update_async(next_segment=seg if i + 1 < K else None)
    ev("after_launch", torch.cuda.current_stream())
    ev("copy_after_prefetch", pipe.copy)
    if pend is not None:
        pend.result()
    pend = h
pend.result()
torch.cuda.synchronize()
ms = (time.perf_counter() - t0) * 1e3 / K
print(f"e2e ms/update {ms:.3f}")
ac = [e for n, e in marks if n == "async_call"]
al = [e for n, e in marks if n == "after_launch"]
cp = [e for n, e in marks if n == "copy_after_prefetch"]
print("compute span launch->launch", [round(al[i].elapsed_time(al[i + 1]), 3) for i in range(len(al) - 1)])
print("copy done rel. to its update's launch end", [round(al[i].elapsed_time(cp[i]), 3) for i in range(len(cp) - 1)])
