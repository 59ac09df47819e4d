"""Graphed cfg2 bf16 update time (device-resident), for A/B of env knobs:
    UL_X=... python tools/step_ablate.py [steps]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_30313_b200 as PKG  # noqa: E402
from paper_2605_30313_b200 import algos as A, tensornet as TN  # noqa: E402
from paper_2605_30313_b200.algos import ppo as P  # noqa: E402
from paper_2605_30313_b200.algos._staging import staging_for  # noqa: E402
from paper_2605_30313_b200.workload import CONFIGS, make_rollout  # noqa: E402

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
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
for _ in range(5):
    try:
        P.ppo_update_resident(ds, params, opt, cfg, rng)
    except Exception:
        pass
torch.cuda.synchronize()
best = []
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        try:
            P.ppo_update_resident(ds, params, opt, cfg, rng)
        except Exception:
            pass
    e1.record()
    torch.cuda.synchronize()
    best.append(e0.elapsed_time(e1) / steps)
print(f"ms/update {min(best):.4f} (reps {' '.join(f'{b:.4f}' for b in best)})")
