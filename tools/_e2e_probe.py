"""Host-side timing of PpoPipeline.update() pieces at cfg2 (diagnostics)."""
import sys, time
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
pipe = A.PpoPipeline(params, opt, cfg, A.DeviceRng(1))
pipe.prefetch(seg)
for _ in range(3):
    pipe.update(next_segment=seg)
torch.cuda.synchronize()
tm = {}
orig = {n: getattr(P, n) for n in ("gae_into", "_launch_epochs", "finish_plan")}
def wrap(n):
    f = orig[n]
    def g(*a, **k):
        t0 = time.perf_counter(); r = f(*a, **k); tm[n] = tm.get(n, 0) + time.perf_counter() - t0; return r
    return g
for n in orig: setattr(P, n, wrap(n))
po = pipe.prefetch
def pf(*a, **k):
    t0 = time.perf_counter(); r = po(*a, **k); tm["prefetch"] = tm.get("prefetch", 0) + time.perf_counter() - t0; return r
pipe.prefetch = pf
K = 10
t0 = time.perf_counter()
for i in range(K):
    pipe.update(next_segment=seg)
torch.cuda.synchronize()
tot = (time.perf_counter() - t0) / K
print("per update ms: total", round(tot * 1e3, 3), {k: round(v / K * 1e3, 3) for k, v in tm.items()})
