"""Measure GPU-vs-oracle parity at the BENCHMARKED shapes (diagnostic, GPU box).

    python tools/parity_probe.py [ppo] [appo] [perf] > gpurun_out/parity_probe.json

ppo : full cfg2 update (24 x 4096, 5 epochs x 4 minibatches) in parity mode
      (reference Philox permutations) for fp32 / tf32 / bf16, against the f32
      oracle (= the reference's arithmetic) and an f64 oracle; also the
      oracle's own f32-vs-f64 gap.
appo: cfg5 shapes at 1/4 size (24 x 4096, obs 98 / 101, act 29).
perf: 3 consecutive bf16 updates, device permutations vs parity mode.
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from threadpoolctl import threadpool_limits  # noqa: E402

threadpool_limits(limits=None)

from oracle import port as O  # noqa: E402
from helpers import _synthetic  # noqa: E402

import paper_2605_30313_b200 as P  # noqa: E402
from paper_2605_30313_b200 import algos as A  # noqa: E402
from paper_2605_30313_b200 import tensornet as TN  # noqa: E402


def to64(n):
    return O.Net(n.dims, [[w.astype(np.float64), b.astype(np.float64)] for w, b in n.layers],
                 n.log_std.astype(np.float64))


def cmp(d_got, d_ref):
    rel = float(np.linalg.norm(d_got - d_ref) / np.linalg.norm(d_ref))
    cos = float(d_got @ d_ref / (np.linalg.norm(d_got) * np.linalg.norm(d_ref)))
    return {"rel": rel, "cos": cos}


def ppo_case(T, N, od, cd, ad, hid, epochs, seed, appo=False, precisions=("fp32", "tf32", "bf16")):
    segd, actor, critic = _synthetic(T, N, od, cd, ad, hid, seed=seed)
    if appo:  # behaviour policy perturbed so ratios != 1
        rng = np.random.default_rng(seed + 100)
        pert = actor.clone()
        for w, b in pert.layers:
            w += rng.normal(0, 1e-3, w.shape).astype(np.float32)
        mean, _ = O.mlp_forward(pert, segd["obs"].reshape(-1, od))
        segd["behavior_log_prob"] = O.gauss_logp(mean, pert.log_std, segd["actions"].reshape(
            -1, ad)).reshape(T, N).astype(np.float64)
    cfg = O.PpoCfg(epochs=epochs)
    out = {"shape": [T, N, od, cd, ad, list(hid)], "epochs": epochs, "appo": appo}
    refs = {}
    for name, conv in (("f32", lambda n: n.clone()), ("f64", to64)):
        a, c = conv(actor), conv(critic)
        oa, oc = O.Opt.for_net(a, cfg.lr), O.Opt.for_net(c, cfg.lr)
        t0 = time.perf_counter()
        if appo:
            sd = dict(segd)
            if name == "f64":
                sd = {k: (v.astype(np.float64) if isinstance(v, np.ndarray) and v.dtype ==
                          np.float32 else v) for k, v in sd.items()}
            st = O.appo_update(sd, a, c, oa, oc, cfg, O.philox_stream(1, "update"))
        else:
            adv, ret = O.gae(segd["rewards"], segd["values"], segd["terminated"],
                             segd["truncated"], segd["bootstrap_value"], 0.99, 0.95,
                             segd["truncation_values"])
            sd = dict(segd, advantages=adv, returns=ret)
            if name == "f64":
                sd = {k: (v.astype(np.float64) if isinstance(v, np.ndarray) and v.dtype ==
                          np.float32 else v) for k, v in sd.items()}
            st = O.ppo_update(sd, a, c, oa, oc, cfg, O.philox_stream(1, "update"))
        refs[name] = (a.flat().astype(np.float64), c.flat().astype(np.float64), st)
        out[f"oracle_{name}_s"] = time.perf_counter() - t0
    a0, c0 = actor.flat().astype(np.float64), critic.flat().astype(np.float64)
    d64 = (refs["f64"][0] - a0, refs["f64"][1] - c0)
    d32 = (refs["f32"][0] - a0, refs["f32"][1] - c0)
    out["oracle_f32_vs_f64"] = {"actor": cmp(d32[0], d64[0]), "critic": cmp(d32[1], d64[1])}
    out["oracle_stats"] = {k: refs["f32"][2][k] for k in ("policy_loss", "value_loss", "kl",
                                                          "grad_norm")}
    for prec in precisions:
        P.set_precision(prec)
        params = A.AcParams(TN.ModelParams.from_numpy(TN.Arch(od, hid, ad), actor.flat()),
                            TN.ModelParams.from_numpy(TN.Arch(cd, hid, 1), critic.flat()))
        seg = A.RolloutSegment(**segd)
        opt = A.AcOpt.for_params(params, 1e-3)
        if appo:
            st = A.appo_update(seg, params, opt, A.AppoConfig(epochs=epochs),
                               O.philox_stream(1, "update"))
        else:
            seg.advantages, seg.returns = A.gae(seg.rewards, seg.values, seg.terminated,
                                                seg.truncated, seg.bootstrap_value, 0.99, 0.95,
                                                truncation_values=seg.truncation_values)
            st = A.ppo_update(seg, params, opt, A.PpoConfig(epochs=epochs),
                              O.philox_stream(1, "update"))
        ga, gc = params.actor.flat().astype(np.float64) - a0, params.critic.flat().astype(
            np.float64) - c0
        out[prec] = {"vs_f32": {"actor": cmp(ga, d32[0]), "critic": cmp(gc, d32[1])},
                     "vs_f64": {"actor": cmp(ga, d64[0]), "critic": cmp(gc, d64[1])},
                     "stats": {"policy_loss": st.policy_loss, "value_loss": st.value_loss,
                               "kl": st.kl, "grad_norm": st.grad_norm}}
        print(json.dumps({prec: out[prec]}), file=sys.stderr, flush=True)
    return out


def perf_case(updates=3):
    """bf16: device permutations vs parity-mode permutations over `updates`."""
    T, N, od, cd, ad, hid = 24, 4096, 235, 235, 12, (512, 256, 128)
    segd, actor, critic = _synthetic(T, N, od, cd, ad, hid, seed=11)
    P.set_precision("bf16")
    res = {}
    for mode in ("parity", "device"):
        params = A.AcParams(TN.ModelParams.from_numpy(TN.Arch(od, hid, ad), actor.flat()),
                            TN.ModelParams.from_numpy(TN.Arch(cd, hid, 1), critic.flat()))
        opt = A.AcOpt.for_params(params, 1e-3)
        rng = O.philox_stream(1, "update") if mode == "parity" else A.DeviceRng(7)
        traj = []
        for u in range(updates):
            seg = A.RolloutSegment(**segd)
            seg.advantages, seg.returns = A.gae(seg.rewards, seg.values, seg.terminated,
                                                seg.truncated, seg.bootstrap_value, 0.99, 0.95,
                                                truncation_values=seg.truncation_values)
            st = A.ppo_update(seg, params, opt, A.PpoConfig(), rng)
            da = params.actor.flat().astype(np.float64) - actor.flat()
            dc = params.critic.flat().astype(np.float64) - critic.flat()
            traj.append({"policy_loss": st.policy_loss, "value_loss": st.value_loss,
                         "kl": st.kl, "grad_norm": st.grad_norm,
                         "dactor": float(np.linalg.norm(da)), "dcritic": float(np.linalg.norm(dc))})
        res[mode] = traj
    return res


def main():
    what = set(sys.argv[1:]) or {"ppo", "appo", "perf"}
    out = {}
    if "ppo" in what:
        out["ppo_cfg2"] = ppo_case(24, 4096, 235, 235, 12, (512, 256, 128), 5, seed=9)
    if "appo" in what:
        out["appo_cfg5_quarter"] = ppo_case(24, 4096, 98, 101, 29, (512, 256, 128), 5, seed=5,
                                            appo=True)
    if "perf" in what:
        out["perf_mode"] = perf_case()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
