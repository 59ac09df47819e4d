"""One cfg2 PPO update (GAE + 5x4 minibatch steps), un-graphed, for ncu launch lists:
    ncu --metrics gpu__time_duration.sum --csv --log-file out.csv python tools/profile_ppo.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_30313_b200 as PKG  # noqa: E402
from paper_2605_30313_b200 import _dev  # noqa: E402
from paper_2605_30313_b200 import algos as A  # noqa: E402
from paper_2605_30313_b200 import tensornet as TN  # noqa: E402
from paper_2605_30313_b200.algos import ppo as P  # noqa: E402
from paper_2605_30313_b200.algos._staging import staging_for  # noqa: E402
from paper_2605_30313_b200.workload import CONFIGS, make_rollout  # noqa: E402

if len(sys.argv) > 1:
    PKG.set_precision(sys.argv[1])
T, N, od, cd, ad, hid = CONFIGS["cfg2"]
cfg = A.PpoConfig()
actor = TN.init_params(TN.Arch(od, hid, ad), 0)
critic = TN.init_params(TN.Arch(cd, hid, 1), 1)
params = A.AcParams(actor, critic)
opt = A.AcOpt.for_params(params, cfg.lr)
w = make_rollout("cfg2", 0)
seg = A.RolloutSegment(obs=w.obs, critic_obs=w.critic_obs, actions=w.actions,
                       behavior_log_prob=np.zeros((T, N)) - 15.0, rewards=w.rewards,
                       terminated=w.terminated, truncated=w.truncated, values=np.zeros((T, N)),
                       bootstrap_value=w.bootstrap_value, truncation_values=w.truncation_values)
ds = staging_for(T, N, od, cd, ad, cfg.epochs)
ds.load(seg, with_advantages=False)
P.gae_into(ds, cfg.gamma, cfg.lam)
P.fill_permutations(ds, A.DeviceRng(1), cfg.epochs)
plan = P._plan_for(params, cfg, ds, 1, 0)
plan.bind(ds, ds.adv, ds.ret, ds.values, params, opt)
torch.cuda.synchronize()
print(P.profile_update(params, opt, cfg, ds))
