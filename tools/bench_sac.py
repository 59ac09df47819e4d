"""cfg3 FastSAC / cfg4 FlashSAC learner benchmark.  cfg3 (BASELINE.json
configs[2]): 2^20-row replay ring resident in HBM as codec rows
(RowCodec(96, 23), 872 B/row), batch 8192 drawn by host indices, twin critics
119->1024->512->256->1 with LayerNorm, actor 96->512->256->128->23,
SacConfig defaults (policy_frequency 4, so one actor/alpha step per 4
updates).  Timed: K sac_update calls (a multiple of 4) with the batch indices
already on the device and device noise (``value``), and the same through host
index vectors + the host noise stream (``e2e``: H2D of 64 KB indices + noise
per update).  CPU baseline: the oracle's sac_update on the same shapes
(--cpu-updates, default 2).  ``--cfg cfg4``: the FlashSAC wide/large-batch
shape of SURVEY.md 8(d) -- batch 32,768, critics 119->1024->1024->1024->1
(no LayerNorm), actor 96->512->512->23, flashsac_defaults (tau 0.01,
policy_frequency 2).  Prints one JSON object.
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_30313_b200 as P  # noqa: E402
from paper_2605_30313_b200 import _dev  # noqa: E402
from paper_2605_30313_b200 import algos as A  # noqa: E402
from paper_2605_30313_b200 import tensornet as TN  # noqa: E402
from paper_2605_30313_b200.algos.ppo import DeviceRng  # noqa: E402

OD, AD, B, RING = 96, 23, 8192, 1 << 20
CH, AH = (1024, 512, 256), (512, 256, 128)
PF = 4  # policy_frequency


def flops_per_update(do_actor: bool) -> float:
    """2 flop/MAC; target fwd (actor + 2 target critics), 2 critic trainings
    (fwd + dW + dH) and, on actor steps, actor fwd + bwd (3x) + 2 critic fwd +
    dH/dX (2x) -- SURVEY.md §8(d) cfg3 row (~14.2 MFLOP/row averaged)."""
    cq = (OD + AD) * CH[0] + sum(CH[i] * CH[i + 1] for i in range(len(CH) - 1)) + CH[-1]
    ca = OD * AH[0] + sum(AH[i] * AH[i + 1] for i in range(len(AH) - 1)) + AH[-1] * AD
    f = 2 * B * (ca + 2 * cq)          # target
    f += 2 * 2 * B * 3 * cq           # critics fwd + dX-free bwd (dW + dH)
    if do_actor:
        f += 2 * B * 3 * ca + 2 * 2 * B * 2 * cq
    return float(f)


def build(ln: bool, flash: bool = False):
    actor = TN.init_params(TN.Arch(OD, AH, AD), 0)
    qa = TN.Arch(OD + AD, CH, 1, layer_norm=ln)
    cfg = A.flashsac_defaults() if flash else A.SacConfig()
    return A.SacState.create(actor, TN.init_params(qa, 1), TN.init_params(qa, 2), cfg), cfg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=8)
    ap.add_argument("--precision", default="bf16")
    ap.add_argument("--no-ln", action="store_true")
    ap.add_argument("--cpu-updates", type=int, default=2)
    ap.add_argument("--cfg", choices=("cfg3", "cfg4"), default="cfg3")
    a = ap.parse_args()
    global B, CH, AH, PF
    if a.cfg == "cfg4":
        B, CH, AH, PF = 32768, (1024, 1024, 1024), (512, 512), 2
        a.no_ln = True
    P.set_precision(a.precision)
    st, cfg = build(not a.no_ln, a.cfg == "cfg4")
    # one learner tick = updates_per_step sac_updates on one batch, one graph
    # launch (R:runtime/sac_runner.py:313-321); cfg4: UTD 8
    utd = 8 if a.cfg == "cfg4" else cfg.updates_per_step
    K = max(1, (a.steps + utd - 1) // utd)
    width = 2 * OD + AD + 3
    g = torch.Generator(device="cuda").manual_seed(0)
    ring = torch.randn(RING, width, device="cuda", generator=g)
    ring[:, OD:OD + AD].tanh_()
    ring[:, 2 * OD + AD + 1] = (torch.rand(RING, device="cuda", generator=g) < 0.01).float()
    ring[:, 2 * OD + AD + 2] = 1.0
    hrng = np.random.default_rng(1)
    idx_dev = [torch.from_numpy(hrng.integers(0, RING, B)).cuda() for _ in range(K)]
    drng = DeviceRng(0)
    s = torch.cuda.current_stream()
    for i in range(max(2, a.warmup // utd)):
        A.sac_updates(A.DeviceRows(ring, width, idx_dev[i % K], B), st, cfg, drng, utd)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.nvtx.range_push("timed")
    e0.record(s)
    for i in range(K):
        A.sac_updates(A.DeviceRows(ring, width, idx_dev[i], B), st, cfg, drng, utd)
    e1.record(s)
    torch.cuda.nvtx.range_pop()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / (K * utd)
    # e2e: host index vector (pinned) + host noise stream each update
    pin = [_dev.pinned_empty((B,), np.int64) for _ in range(2)]
    idx_buf = torch.empty(B, dtype=torch.int64, device="cuda")
    host_rng = np.random.default_rng(2)
    nrng = np.random.default_rng(3)

    def e2e_step(i, noise):
        h = pin[i & 1]
        h[:] = host_rng.integers(0, RING, B)
        idx_buf.copy_(torch.from_numpy(h), non_blocking=True)
        return A.sac_updates(A.DeviceRows(ring, width, idx_buf, B), st, cfg, noise, utd)[-1]

    def e2e(noise):
        for i in range(4):
            e2e_step(i, noise)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(K):
            last = e2e_step(i, noise)
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) * 1e3 / (K * utd), last

    # performance mode (device Philox noise) and parity mode (the reference's
    # host standard_normal stream: B x A normals twice per update on the host)
    e2e_ms, out = e2e(drng)
    e2e_parity_ms, _ = e2e(nrng)
    fl = ((PF - 1) * flops_per_update(False) + flops_per_update(True)) / PF
    res = {
        "workload": f"{a.cfg} {'FlashSAC' if a.cfg == 'cfg4' else 'FastSAC'} sac_update (ring 2^20 x "
                    f"RowCodec(96,23), batch {B}, critics 119-{'-'.join(map(str, CH))}-1"
                    f"{' +LN' if not a.no_ln else ''}, actor 96-{'-'.join(map(str, AH))}-23,"
                    f" policy_frequency {PF})",
        "precision": a.precision, "updates": K * utd, "updates_per_tick": utd,
        "graph": "one CUDA graph launch per tick (sac_updates)",
        "ms_per_update": ms, "updates_per_s": 1e3 / ms,
        "e2e_ms_per_update": e2e_ms, "e2e_updates_per_s": 1e3 / e2e_ms,
        "e2e": "host batch indices each tick (pinned H2D), device noise, one graph per tick",
        "e2e_parity_mode_ms_per_update": e2e_parity_ms,
        "tflops_achieved": fl / (ms * 1e-3) / 1e12,
        "critic_loss_last": out.extra["critic_loss"],
    }
    if a.cpu_updates > 0:
        from oracle import port as O
        ost = O.SacSt.create(O.net_init((OD, *AH, AD), 0),
                             O.net_init((OD + AD, *CH, 1), 1, layer_norm=not a.no_ln),
                             O.net_init((OD + AD, *CH, 1), 2, layer_norm=not a.no_ln),
                             O.SacCfg(policy_frequency=1))
        ocfg = O.SacCfg(policy_frequency=1)
        ring_h = ring[:B * 2].cpu().numpy()
        from paper_2605_30313_b200.replaypath.storage import RowCodec
        batch = RowCodec(OD, AD).decode(ring_h[:B])
        r = np.random.default_rng(0)
        O.sac_update(batch, ost, O.SacCfg(policy_frequency=4), r)  # warm (critic only)
        t0 = time.perf_counter()
        for _ in range(a.cpu_updates):  # every update with the actor step: upper bound
            O.sac_update(batch, ost, ocfg, r)
        cpu_s = (time.perf_counter() - t0) / a.cpu_updates
        import os
        res["cpu_baseline"] = {"ms_per_update_with_actor": cpu_s * 1e3,
                               "cores": len(os.sched_getaffinity(0)), "kind": "port",
                               "sample": f"{a.cpu_updates} oracle sac_update calls, actor step "
                                         "each (policy_frequency 1)"}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
