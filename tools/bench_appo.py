"""cfg5 APPO learner benchmark (BASELINE.json configs[4], SURVEY.md 8(d) cfg5
row): T = 24 x N = 16,384 envs of the G1 humanoid shape (obs 98 / critic obs
101 / 29 actions), actor + critic 512-256-128, AppoConfig defaults; behavior
log-probs from parameters perturbed by N(0, 1e-3) so the V-trace ratios are
not 1.  One step = ``appo_update`` on a segment resident in HBM: recompute
target log-probs and values over all 393,216 rows, V-trace (K2), then
5 epochs x 4 minibatches of 98,304 rows.  CUDA events over K steps.  CPU
baseline: the oracle's appo_update on a bounded sample (N_cpu envs, 1 epoch)
extrapolated to the full update.  Prints one JSON object.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_30313_b200 as P  # noqa: E402
from paper_2605_30313_b200 import algos as A  # noqa: E402
from paper_2605_30313_b200 import tensornet as TN  # noqa: E402
from paper_2605_30313_b200.algos import appo as AP  # noqa: E402
from paper_2605_30313_b200.algos._staging import staging_for  # noqa: E402
from paper_2605_30313_b200.workload import CONFIGS, make_rollout  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--precision", default="bf16")
    ap.add_argument("--cpu-envs", type=int, default=1024)
    a = ap.parse_args()
    P.set_precision(a.precision)
    T, N, od, cd, ad, hid = CONFIGS["cfg5"]
    cfg = A.AppoConfig()
    actor = TN.init_params(TN.Arch(od, hid, ad), 0)
    critic = TN.init_params(TN.Arch(cd, hid, 1), 1)
    params = A.AcParams(actor, critic)
    opt = A.AcOpt.for_params(params, cfg.lr)
    w = make_rollout("cfg5", 0)
    rng = np.random.default_rng(5)
    # behavior policy = actor perturbed by N(0, 1e-3): log-probs from the oracle math on host
    from oracle import port as O
    ba = O.net_init((od, *hid, ad), 0)
    ba = O.Net(ba.dims, [[wt + 1e-3 * rng.standard_normal(wt.shape).astype(np.float32),
                          b + 1e-3 * rng.standard_normal(b.shape).astype(np.float32)]
                         for wt, b in ba.layers], ba.log_std)
    flat = lambda x: x.reshape(-1, x.shape[-1])  # noqa: E731
    mean, _ = O.mlp_forward(ba, flat(w.obs))
    blogp = O.gauss_logp(mean, ba.log_std, flat(w.actions)).reshape(T, N)
    seg = A.RolloutSegment(obs=w.obs, critic_obs=w.critic_obs, actions=w.actions,
                           behavior_log_prob=blogp, rewards=w.rewards, terminated=w.terminated,
                           truncated=w.truncated, values=np.zeros((T, N)),
                           bootstrap_value=w.bootstrap_value,
                           truncation_values=w.truncation_values)
    ds = staging_for(T, N, od, cd, ad, cfg.epochs, slot="appo")
    ds.load(seg, with_advantages=False)
    drng = A.DeviceRng(1)
    for _ in range(a.warmup):
        AP.appo_update_resident(ds, params, opt, cfg, drng)
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(a.steps):
        st = AP.appo_update_resident(ds, params, opt, cfg, drng)
    e1.record(s)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    # the recompute forward (target log-prob + V(s) of the whole segment) and
    # V-trace alone, for the phase split
    e0.record(s)
    for _ in range(a.steps):
        AP.recompute_targets(ds, params)
        AP.vtrace_into(ds, cfg)
    e1.record(s)
    e1.synchronize()
    rec_ms = e0.elapsed_time(e1) / a.steps
    rows = T * N
    res = {"workload": "cfg5 APPO appo_update (V-trace), 24 x 16384 envs, obs 98 / cobs 101 / "
                       "act 29, actor+critic 512-256-128, 5 epochs x 4 minibatches, segment "
                       "resident in HBM, device minibatch permutations",
           "precision": a.precision, "steps": a.steps, "ms_per_update": ms,
           "recompute_vtrace_ms": rec_ms,
           "transitions_per_s": rows / (ms * 1e-3), "policy_loss_last": st.policy_loss}
    # CPU: the oracle appo_update on cpu_envs envs, 1 epoch, extrapolated
    n = a.cpu_envs
    if n <= 0:
        print(json.dumps(res))
        return
    sub = {k: v[:, :n] for k, v in dict(obs=w.obs, critic_obs=w.critic_obs, actions=w.actions,
                                        behavior_log_prob=blogp.astype(np.float64),
                                        rewards=w.rewards, terminated=w.terminated,
                                        truncated=w.truncated,
                                        truncation_values=w.truncation_values).items()}
    sub["values"] = np.zeros((T, n))
    sub["bootstrap_value"] = w.bootstrap_value[:n]
    oa_net, oc_net = O.net_init((od, *hid, ad), 0), O.net_init((cd, *hid, 1), 1)
    ocfg = O.PpoCfg(epochs=1)
    oa, oc = O.Opt.for_net(oa_net, ocfg.lr), O.Opt.for_net(oc_net, ocfg.lr)
    t0 = time.perf_counter()
    O.appo_update(sub, oa_net, oc_net, oa, oc, ocfg, O.philox_stream(1, "update"))
    spent = time.perf_counter() - t0
    # the epoch loop dominates; scale rows x epochs (recompute/V-trace scale with rows only)
    cpu_ms = spent * (N / n) * 5.0 * 1e3
    res["cpu_baseline"] = {"ms_per_update": cpu_ms, "transitions_per_s": rows / (cpu_ms * 1e-3),
                           "cores": len(os.sched_getaffinity(0)), "kind": "port",
                           "sample": f"oracle appo_update on {n} of {N} envs, 1 of 5 epochs, "
                                     "extrapolated x(N/n) x5 (an upper bound: recompute and "
                                     "V-trace do not repeat per epoch)",
                           "seconds": spent}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
