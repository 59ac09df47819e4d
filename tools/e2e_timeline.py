"""Device timeline of the async e2e loop (PpoPipeline.update_async, cfg2): per update, the copy-stream H2D
duration and the compute-stream span, and the gap between updates."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_2605_30313_b200 as PKG
from paper_2605_30313_b200 import algos as A, tensornet as TN, _dev
from paper_2605_30313_b200.algos import ppo as P
from paper_2605_30313_b200.workload import CONFIGS, make_rollout
PKG.set_precision("bf16")
T, N, od, cd, ad, hid = CONFIGS["cfg2"]
cfg = A.PpoConfig()
params = A.AcParams(TN.init_params(TN.Arch(od, hid, ad), 0), TN.init_params(TN.Arch(cd, hid, 1), 1))
opt = A.AcOpt.for_params(params, cfg.lr)
w = make_rollout("cfg2", 0)
def pin(a):
    b = _dev.pinned_empty(a.shape, a.dtype); b[...] = a; return b
seg = A.RolloutSegment(obs=pin(w.obs), critic_obs=pin(w.critic_obs), actions=pin(w.actions),
                       behavior_log_prob=pin(np.zeros((T, N)) - 15.0), rewards=pin(w.rewards),
                       terminated=pin(w.terminated), truncated=pin(w.truncated), values=pin(np.zeros((T, N))),
                       bootstrap_value=pin(w.bootstrap_value), truncation_values=pin(w.truncation_values))
mode = sys.argv[1] if len(sys.argv) > 1 else "full"
pipe = A.PpoPipeline(params, opt, cfg, A.DeviceRng(1))
ev = []
po = pipe.prefetch
def pf(segment):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(pipe.copy)
    if mode == "nocopy" and pipe.slots[pipe.next_slot] is not None:
        # stage nothing new: re-queue the slot as if loaded
        k = pipe.next_slot; pipe.next_slot ^= 1
        pipe.copy.wait_event(pipe.free[k]); pipe.ready[k].record(pipe.copy); pipe.queue.append(k)
    else:
        po(segment)
    b.record(pipe.copy)
    ev.append(("copy", a, b))
pipe.prefetch = pf
ol = P._launch_epochs
def le(*a, **k):
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s); r = ol(*a, **k); e1.record(s)
    ev.append(("upd", e0, e1)); return r
P._launch_epochs = le
pipe.prefetch(seg)
for _ in range(3):
    pipe.update(next_segment=seg)
torch.cuda.synchronize()
ev.clear()
import time
HT = {}
def htime(name, f):
    def g(*a, **k):
        t = time.perf_counter(); r = f(*a, **k); HT[name] = HT.get(name, 0) + time.perf_counter() - t; return r
    return g
P.gae_into = htime("gae_into", P.gae_into)
P._launch_epochs = htime("_launch_epochs", P._launch_epochs)
P.fill_permutations = htime("fill_perm", P.fill_permutations)
P.launch_plan = htime("launch_plan", P.launch_plan)
P._drain_pending = htime("drain", P._drain_pending)
pipe.prefetch = htime("prefetch", pipe.prefetch)
K = 12
t0 = time.perf_counter()
pend = None
hu, hr = [], []
for i in range(K):
    t1 = time.perf_counter()
    h = pipe.update_async(next_segment=seg if i + 1 < K else None)
    t2 = time.perf_counter()
    if pend is not None:
        pend.result()
    hu.append(t2 - t1); hr.append(time.perf_counter() - t2)
    pend = h
pend.result()
torch.cuda.synchronize()
tot = (time.perf_counter() - t0) / K * 1e3
ups = [(a, b) for n, a, b in ev if n == "upd"]
cps = [(a, b) for n, a, b in ev if n == "copy"]
print(mode, "e2e ms/update", round(tot, 3))
print("host update_async ms", [round(x * 1e3, 3) for x in hu])
print("host result ms", [round(x * 1e3, 3) for x in hr])
print("host phase ms/iter", {k: round(v / K * 1e3, 3) for k, v in HT.items()})
print("update spans", [round(a.elapsed_time(b), 3) for a, b in ups])
print("copy spans", [round(a.elapsed_time(b), 3) for a, b in cps])
print("gaps upd_end->next upd_start", [round(ups[i][1].elapsed_time(ups[i + 1][0]), 3) for i in range(len(ups) - 1)])
