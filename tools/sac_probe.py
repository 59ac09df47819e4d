"""SAC parity at the benchmarked shapes (diagnostic, GPU box).

    python tools/sac_probe.py [cfg3] [cfg4] > gpurun_out/sac_probe.json

Runs U consecutive sac_update calls (reference noise stream, host batch) on
the GPU for fp32 / tf32 / bf16 and on the oracle in f32 and f64; reports
per-network parameter-delta rel / cos against f64 and the loss trajectories.
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from threadpoolctl import threadpool_limits  # noqa: E402

threadpool_limits(limits=None)

from oracle import port as O  # noqa: E402

import paper_2605_30313_b200 as P  # noqa: E402
from paper_2605_30313_b200 import algos as A  # noqa: E402
from paper_2605_30313_b200 import tensornet as TN  # noqa: E402

CFGS = {
    # name: (obs, act, critic hidden, actor hidden, LN, batch, flash, updates)
    "cfg3": (96, 23, (1024, 512, 256), (512, 256, 128), True, 8192, False, 4),
    "cfg4": (96, 23, (1024, 1024, 1024), (512, 512), False, 32768, True, 4),
}


def to64(n):
    return O.Net(n.dims, [[w.astype(np.float64), b.astype(np.float64)] for w, b in n.layers],
                 n.log_std.astype(np.float64),
                 [[g.astype(np.float64), b.astype(np.float64)] for g, b in n.ln])


def cmp(d, r):
    return {"rel": float(np.linalg.norm(d - r) / np.linalg.norm(r)),
            "cos": float(d @ r / (np.linalg.norm(d) * np.linalg.norm(r)))}


def batch_of(B, od, ad, seed):
    rng = np.random.default_rng(seed)
    return dict(obs=rng.normal(size=(B, od)).astype(np.float32),
                action=np.tanh(rng.normal(size=(B, ad))).astype(np.float32),
                reward=rng.normal(size=B).astype(np.float32),
                next_obs=rng.normal(size=(B, od)).astype(np.float32),
                terminated=rng.random(B) < 0.01, n_used=np.ones(B, np.int64))


def case(name):
    od, ad, ch, ah, ln, B, flash, U = CFGS[name]
    a0 = O.net_init((od, *ah, ad), 0)
    q0 = [O.net_init((od + ad, *ch, 1), s, layer_norm=ln) for s in (1, 2)]
    cfg = A.flashsac_defaults() if flash else A.SacConfig()
    ocfg = O.SacCfg(tau=cfg.tau, policy_frequency=cfg.policy_frequency)
    batch = batch_of(B, od, ad, 3)
    out = {"shape": CFGS[name]}
    refs = {}
    for kind, conv in (("f32", lambda n: n.clone()), ("f64", to64)):
        st = O.SacSt.create(conv(a0), conv(q0[0]), conv(q0[1]), ocfg)
        bt = batch if kind == "f32" else {k: (v.astype(np.float64) if v.dtype == np.float32
                                             else v) for k, v in batch.items()}
        rng = O.philox_stream(1, "learner")
        t0 = time.perf_counter()
        traj = [O.sac_update(bt, st, ocfg, rng) for _ in range(U)]
        out[f"oracle_{kind}_s"] = time.perf_counter() - t0
        refs[kind] = (st, traj)
    init = {"actor": a0.flat(), "q1": q0[0].flat(), "q2": q0[1].flat()}
    d = {k: {n: getattr(refs[k][0], n).flat().astype(np.float64) - init[n] for n in init}
         for k in refs}
    out["oracle_f32_vs_f64"] = {n: cmp(d["f32"][n], d["f64"][n]) for n in init}
    out["oracle_traj"] = refs["f32"][1]
    qa = TN.Arch(od + ad, ch, 1, layer_norm=ln)
    for prec in ("fp32", "tf32", "bf16"):
        P.set_precision(prec)
        st = A.SacState.create(TN.ModelParams.from_numpy(TN.Arch(od, ah, ad), a0.flat()),
                               TN.ModelParams.from_numpy(qa, q0[0].flat()),
                               TN.ModelParams.from_numpy(qa, q0[1].flat()), cfg)
        rng = O.philox_stream(1, "learner")
        stats = A.sac_updates(batch, st, cfg, rng, U)
        got = {"actor": st.params.actor.flat(), "q1": st.params.q1.flat(),
               "q2": st.params.q2.flat()}
        res = {"vs_f64": {n: cmp(got[n].astype(np.float64) - init[n], d["f64"][n]) for n in init},
               "vs_f32": {n: cmp(got[n].astype(np.float64) - init[n], d["f32"][n]) for n in init},
               "traj": [s.extra for s in stats], "log_alpha": st.params.log_alpha,
               "oracle_log_alpha": refs["f32"][0].log_alpha}
        # the one-graph run equals U separate calls, bit for bit
        st2 = A.SacState.create(TN.ModelParams.from_numpy(TN.Arch(od, ah, ad), a0.flat()),
                                TN.ModelParams.from_numpy(qa, q0[0].flat()),
                                TN.ModelParams.from_numpy(qa, q0[1].flat()), cfg)
        rng2 = O.philox_stream(1, "learner")
        for _ in range(U):
            A.sac_update(batch, st2, cfg, rng2)
        res["graph_equals_sequential"] = bool(
            np.array_equal(st2.params.q1.flat(), got["q1"])
            and np.array_equal(st2.params.actor.flat(), got["actor"])
            and np.array_equal(st2.params.q2_targ.flat(), st.params.q2_targ.flat()))
        out[prec] = res
        print(json.dumps({name: {prec: {k: res[k] for k in ("vs_f64", "graph_equals_sequential")}}}),
              file=sys.stderr, flush=True)
    return out


def main():
    what = sys.argv[1:] or ["cfg3", "cfg4"]
    print(json.dumps({w: case(w) for w in what}, indent=1, default=float))


if __name__ == "__main__":
    main()
