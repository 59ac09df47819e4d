#!/usr/bin/env python
"""Learner throughput of the PPO locomotion-shape update (BASELINE.json configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one learner iteration of R:runtime/ppo_runner.py:95-104 on a
synthetic cfg2 rollout (T=24 x N=4096 envs, obs = critic_obs = 235, act 12,
actor/critic 512-256-128, PpoConfig defaults: 5 epochs x 4 minibatches):
GAE + ppo_update.

  value  device-resident: the segment is already in HBM; K x (GAE kernel +
         the update plan replayed as one CUDA graph), CUDA events, max over
         ranks.  Minibatch indices: device permutation ("performance mode").
  e2e    through the public pipeline API (algos.PpoPipeline.update_async:
         double-buffered pinned-host -> HBM staging ring, GAE on the device,
         statistics read one update behind) from pinned HOST buffers: every
         step H2D of the whole segment (~192 MB), the update, and the D2H of
         the update's result record.  The serial reference-signature flow
         (algos.gae + algos.ppo_update per step) is reported beside it.
  tf32_arm  the same update with tf32 tensor-core GEMMs (same-width check
         next to the bf16 headline).
Multi-GPU (torchrun): one process per GPU, NCCL all-reduce of the gradient
buffer every minibatch step.  --scaling weak (default): every rank owns its
own 4096-env segment, value = (N x 98,304 transitions) / max-over-ranks step
time.  --scaling strong: one 4096-env segment replicated on every rank, each
rank takes 1/N of every minibatch (value = 98,304 / step time).

``--impl reference`` times the reference's own CPU learner: the UNMODIFIED
reference package installed into baseline/_ref (pip --target), called through
its public API (unilite.algos.gae + unilite.algos.ppo_update, reference Philox
update stream) on every host core, whole learner iterations (not
extrapolated); the numpy oracle port is used only if baseline/_ref is absent.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "learner transitions/sec at 1/2/4/8 B200 vs host-CPU ref; PPO update ms/iter"
UNIT = "transitions/s"
CFG = "cfg2"


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--precision", choices=("fp32", "tf32", "bf16"), default="bf16")
    ap.add_argument("--ref-budget", type=float, default=60.0,
                    help="seconds of timed reference updates (--impl reference)")
    ap.add_argument("--scaling", choices=("weak", "strong"), default="weak")
    return ap.parse_args()


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d["hbm_gbs"], d["bf16_tflops"], d["bf16_tflops_sustained"], "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi-equivalent sampling (NVML) of SM clocks / throttle reasons
    during the timed region."""

    def __init__(self, index: int):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if mask & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            self._stop.wait(0.01)  # (the timed region is ~0.1 s: sample every 10 ms)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=2)

    def summary(self):
        med = float(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# --------------------------------------------------------- CPU reference arm
REF_DIR = ROOT / "baseline" / "_ref"  # unmodified reference package (pip --target install)


def _cpu_threads(n=None):
    """Limit BLAS/OpenMP pools to n threads (default: every host core)."""
    from threadpoolctl import threadpool_limits

    n = n or os.cpu_count() or 1
    return threadpool_limits(limits=n), n


def _reference_pkg():
    """The unmodified reference (``unilite``) from baseline/_ref, or None."""
    if not (REF_DIR / "unilite").is_dir():
        return None
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    import unilite  # noqa: F401
    import unilite.algos
    import unilite.envcore.rng
    import unilite.tensornet

    return unilite


class RefLearner:
    """The reference's own CPU learner step on the cfg2 workload, through its
    public API: ``gae`` + ``ppo_update`` (R:runtime/ppo_runner.py:95-102) with
    the reference update stream ``stream(1, "update")``.  Falls back to the
    numpy oracle port (kind "port") only when baseline/_ref is absent."""

    def __init__(self, seed: int = 0):
        from paper_2605_30313_b200.workload import CONFIGS, make_rollout

        T, N, od, cd, ad, hid = CONFIGS[CFG]
        self.T, self.N = T, N
        w = make_rollout(CFG, seed)
        U = _reference_pkg()
        self.kind = "reference" if U is not None else "port"
        flat = lambda a: a.reshape(-1, a.shape[-1])
        if U is not None:
            TN, AL = U.tensornet, U.algos
            actor = TN.init_params(TN.Arch(od, hid, ad), 0)
            critic = TN.init_params(TN.Arch(cd, hid, 1), 1)
            mean, _ = TN.forward(actor, flat(w.obs))
            blogp = TN.gaussian_log_prob(mean, actor.log_std, flat(w.actions))
            vals, _ = TN.value_forward(critic, flat(w.critic_obs))
            self.seg = AL.RolloutSegment(
                obs=w.obs, critic_obs=w.critic_obs, actions=w.actions,
                behavior_log_prob=np.asarray(blogp, np.float64).reshape(T, N),
                rewards=w.rewards, terminated=w.terminated, truncated=w.truncated,
                values=np.asarray(vals, np.float64).reshape(T, N),
                bootstrap_value=w.bootstrap_value, truncation_values=w.truncation_values)
            self.params = AL.AcParams(actor, critic)
            self.cfg = AL.PpoConfig()
            self.opt = AL.AcOpt.for_params(self.params, self.cfg.lr)
            self.rng = U.envcore.rng.stream(1, "update")
            self.U = U
        else:
            from oracle import port as O

            actor = O.net_init((od, *hid, ad), 0)
            critic = O.net_init((cd, *hid, 1), 1)
            mean, _ = O.mlp_forward(actor, flat(w.obs))
            blogp = O.gauss_logp(mean, actor.log_std, flat(w.actions)).reshape(T, N)
            vals = O.value_forward(critic, flat(w.critic_obs))[0].reshape(T, N)
            self.seg = dict(obs=w.obs, critic_obs=w.critic_obs, actions=w.actions,
                            behavior_log_prob=blogp.astype(np.float64), rewards=w.rewards,
                            terminated=w.terminated, truncated=w.truncated,
                            values=vals.astype(np.float64), bootstrap_value=w.bootstrap_value,
                            truncation_values=w.truncation_values)
            self.actor, self.critic = actor, critic
            self.cfg = O.PpoCfg()
            self.oa, self.oc = O.Opt.for_net(actor, self.cfg.lr), O.Opt.for_net(critic, self.cfg.lr)
            self.rng = O.philox_stream(1, "update")
            self.O = O

    def step(self, epochs: int | None = None) -> float:
        """One learner iteration (GAE + the full update, or its first
        `epochs` epochs); returns seconds."""
        t0 = time.perf_counter()
        if self.kind == "reference":
            AL = self.U.algos
            s = self.seg
            s.advantages, s.returns = AL.gae(s.rewards, s.values, s.terminated, s.truncated,
                                             s.bootstrap_value, self.cfg.gamma, self.cfg.lam,
                                             truncation_values=s.truncation_values)
            cfg = self.cfg if epochs is None else AL.PpoConfig(epochs=epochs)
            AL.ppo_update(s, self.params, self.opt, cfg, self.rng)
        else:
            O, s = self.O, self.seg
            adv, ret = O.gae(s["rewards"], s["values"], s["terminated"], s["truncated"],
                             s["bootstrap_value"], 0.99, 0.95, s["truncation_values"])
            cfg = self.cfg if epochs is None else O.PpoCfg(epochs=epochs)
            O.ppo_update(dict(s, advantages=adv, returns=ret), self.actor, self.critic, self.oa,
                         self.oc, cfg, self.rng)
        return time.perf_counter() - t0


def cpu_reference_run(steps: int, warmup: int, budget_s: float, seed: int = 0):
    """Whole reference learner iterations on every host core: `warmup`
    untimed, then up to `steps` timed, stopping once `budget_s` seconds of
    timed work have run (at least one).  Also a 1-thread reading on a
    bounded sample (GAE + 1 of 5 epochs, x5).  Returns a dict."""
    ref = RefLearner(seed)
    lim, cores = _cpu_threads()
    for _ in range(warmup):
        ref.step()
    times = []
    while len(times) < steps:
        times.append(ref.step())
        if sum(times) >= budget_s:
            break
    lim1, _ = _cpu_threads(1)
    one = ref.step(epochs=1)
    _cpu_threads()
    update_s = float(np.median(times))
    return {"kind": ref.kind, "cores": cores, "steps_run": len(times), "update_ms": update_s * 1e3,
            "value": ref.T * ref.N / update_s, "seconds": float(sum(times)),
            "threads_1": {"update_ms_est": one * 5e3, "value": ref.T * ref.N / (one * 5),
                          "sample": "GAE + 1 of 5 epochs at 1 BLAS thread, x5"}}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    t0 = time.perf_counter()
    r = cpu_reference_run(args.steps, min(args.warmup, 1), budget_s=args.ref_budget)
    wall = time.perf_counter() - t0
    src = ("unmodified reference package (baseline/_ref/unilite): unilite.algos.gae + "
           "unilite.algos.ppo_update" if r["kind"] == "reference"
           else "numpy oracle port of R:algos/estimators.py + R:algos/ppo.py")
    sample = (f"{r['steps_run']} whole cfg2 learner iterations (GAE + ppo_update, 5 epochs x 4 "
              f"minibatches of 24,576 rows), median; {src}; {r['cores']} BLAS threads")
    line = {"impl": "reference", "metric": METRIC, "value": r["value"], "unit": UNIT,
            "n_gpus": args.gpus, "steps": r["steps_run"], "steps_requested": args.steps,
            "warmup": min(args.warmup, 1), "ms_per_step": r["update_ms"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32 networks / f64 estimators+loss (reference numpy)", "data": "synthetic",
            "config": {"workload": "PPO update, cfg2 locomotion shape (4096 envs x 24, obs 235, "
                                   "act 12, 512-256-128, 5x4 minibatches)",
                       "global_batch": 98304, "parallelism": "host CPU",
                       "indices": "reference Philox stream(1, 'update')"},
            "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": r["cores"],
                             "kind": r["kind"], "sample": sample,
                             "threads_1": r["threads_1"]},
            "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "wall_s": wall}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2605_30313_b200 import _dev, _dist
    from paper_2605_30313_b200 import algos as A
    from paper_2605_30313_b200 import tensornet as TN
    from paper_2605_30313_b200.algos import ppo as P
    from paper_2605_30313_b200.algos._staging import staging_for
    from paper_2605_30313_b200.workload import CONFIGS, make_rollout

    import paper_2605_30313_b200 as PKG

    if args.precision:
        PKG.set_precision(args.precision)
    prec = PKG.get_precision()
    prec_name = {"fp32": "fp32 SIMT FFMA", "tf32": "tcgen05 kind::tf32 (TMA + TMEM)",
                 "bf16": "tcgen05 kind::f16 bf16 operands, fp32 accumulation (TMA + TMEM)"}[prec]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    if world > 1:
        # UL_DIST_BACKEND=gloo: a functional check of the multi-rank path when
        # the ranks must share one GPU (NCCL refuses duplicate devices)
        backend = os.environ.get("UL_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        _dist.set_segment_mode("local" if args.scaling == "weak" else "replicated")
    strong = args.scaling == "strong" and world > 1
    seed_rank = 0 if strong else rank  # strong scaling: one replicated segment / stream
    T, N, od, cd, ad, hid = CONFIGS[CFG]
    cfg = A.PpoConfig()

    # networks (reference init, seeds 0 / 1) and a pinned host rollout per rank
    actor = TN.init_params(TN.Arch(od, hid, ad), 0)
    critic = TN.init_params(TN.Arch(cd, hid, 1), 1)
    params = A.AcParams(actor, critic)
    opt = A.AcOpt.for_params(params, cfg.lr)
    w = make_rollout(CFG, seed=seed_rank, alloc=_dev.pinned_empty)
    # behaviour log-prob and values at init, computed by our own kernels
    mean, _ = TN.forward(actor, w.obs.reshape(-1, od))
    blogp = TN.gaussian_log_prob(mean, actor.log_std, w.actions.reshape(-1, ad))
    vals, _ = TN.value_forward(critic, w.critic_obs.reshape(-1, cd))
    w.behavior_log_prob = _dev.pinned_empty((T, N), np.float64)
    w.behavior_log_prob[...] = blogp.cpu().numpy().reshape(T, N)
    w.values = _dev.pinned_empty((T, N), np.float64)
    w.values[...] = vals.cpu().numpy().reshape(T, N)
    seg = A.RolloutSegment(obs=w.obs, critic_obs=w.critic_obs, actions=w.actions,
                           behavior_log_prob=w.behavior_log_prob, rewards=w.rewards,
                           terminated=w.terminated, truncated=w.truncated, values=w.values,
                           bootstrap_value=w.bootstrap_value, truncation_values=w.truncation_values)

    ds = staging_for(T, N, od, cd, ad, cfg.epochs)
    ds.load(seg, with_advantages=False)
    rng = A.DeviceRng(seed=1000 + seed_rank)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident learner steps (value)
    for _ in range(args.warmup):
        P.ppo_update_resident(ds, params, opt, cfg, rng)
    torch.cuda.synchronize()
    smi = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with smi:
        e0.record()
        for _ in range(args.steps):
            P.ppo_update_resident(ds, params, opt, cfg, rng)
        e1.record()
        torch.cuda.synchronize()
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1)) / args.steps
    transitions = (1 if strong else world) * T * N
    value = transitions / (ms / 1e3)

    # ---- parity mode: the reference's own host Philox permutations
    from paper_2605_30313_b200.algos.ppo import fill_permutations  # noqa: F401

    prng = np.random.Generator(np.random.Philox(key=1234 + seed_rank))
    P.ppo_update_resident(ds, params, opt, cfg, prng)
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    n_par = 3
    for _ in range(n_par):
        P.ppo_update_resident(ds, params, opt, cfg, prng)
    torch.cuda.synchronize()
    par_ms = max_over_ranks((time.perf_counter() - t0) * 1e3 / n_par)

    # host cost of the reference's index stream alone (SURVEY.md 7 hard part
    # 10): cfg.epochs Philox permutations of the update's rows
    t0 = time.perf_counter()
    hr = np.random.Generator(np.random.Philox(key=7))
    for _ in range(cfg.epochs):
        hr.permutation(T * N)
    host_perm_ms = (time.perf_counter() - t0) * 1e3

    # ---- other GEMM back ends on the identical update: tf32 (same-width
    # check next to the bf16 headline) and 3xTF32 (the fp32-parity
    # precision on the tensor cores); device permutations, CUDA events
    arms = {}
    arm_desc = {"tf32": "tcgen05 kind::tf32 (fp32 storage, activations and accumulation)",
                "tf32x3": "tcgen05 kind::tf32 over 3xTF32-split fp32 operands (fp32 parity: "
                          "hi*hi + hi*lo + lo*hi as one GEMM over a tripled K)"}
    for arm in ("tf32", "tf32x3"):
        if arm == prec:
            continue
        PKG.set_precision(arm)
        # (the bf16 headline stages bf16 observation rows; an fp32-storage
        # back end gets its own fp32 staging of the same segment)
        ds_arm = staging_for(T, N, od, cd, ad, cfg.epochs)
        ds_arm.load(seg, with_advantages=False)
        for _ in range(2):
            P.ppo_update_resident(ds_arm, params, opt, cfg, rng)
        torch.cuda.synchronize()
        barrier()
        t0e, t1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n_arm = max(3, min(args.steps, 10)) if arm == "tf32" else 3
        t0e.record()
        for _ in range(n_arm):
            P.ppo_update_resident(ds_arm, params, opt, cfg, rng)
        t1e.record()
        torch.cuda.synchronize()
        a_ms = max_over_ranks(t0e.elapsed_time(t1e)) / n_arm
        arms[arm] = {"value": transitions / (a_ms / 1e3), "unit": UNIT, "update_ms": a_ms,
                     "steps": n_arm, "gemm_precision": arm_desc[arm]}
        PKG.set_precision(prec)
    tf32 = arms.get("tf32")

    # ---- e2e through the public API from pinned host buffers: the
    # double-buffered staging pipeline (segment i+1's H2D overlaps update i;
    # update i+1 is enqueued, device-chained, before update i's statistics
    # are read; every step's H2D and its stats D2H are inside the timed region)
    # (a steady-state run: the first segment's copy has no earlier update to
    # hide behind, so it is amortised over at least 50 updates, as in a
    # learner that runs for many iterations; every step still carries one
    # full segment H2D and a stats D2H)
    e2e_steps = args.e2e_steps or max(50, args.steps)
    pipe = A.PpoPipeline(params, opt, cfg, rng)
    for _ in range(2):
        pipe.prefetch(seg)
        pipe.update()
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    pipe.prefetch(seg)
    pend = None
    for i in range(e2e_steps):
        h = pipe.update_async(next_segment=seg if i + 1 < e2e_steps else None)
        if pend is not None:
            st = pend.result()  # update i-1's host stats (D2H) while update i runs
        pend = h
    st = pend.result()
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks((time.perf_counter() - t0) * 1e3 / e2e_steps)
    h2d = ds.h2d_bytes(seg, with_advantages=False)
    d2h = 8 * 9 + 8 * 3  # ul_ppo_result + stats

    # serial reference flow for comparison: host-facing gae + ppo_update
    for _ in range(1):
        seg.advantages, seg.returns = A.gae(seg.rewards, seg.values, seg.terminated,
                                            seg.truncated, seg.bootstrap_value, cfg.gamma,
                                            cfg.lam, truncation_values=seg.truncation_values)
        A.ppo_update(seg, params, opt, cfg, rng)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        seg.advantages, seg.returns = A.gae(seg.rewards, seg.values, seg.terminated,
                                            seg.truncated, seg.bootstrap_value, cfg.gamma,
                                            cfg.lam, truncation_values=seg.truncation_values)
        A.ppo_update(seg, params, opt, cfg, rng)
    torch.cuda.synchronize()
    serial_ms = max_over_ranks((time.perf_counter() - t0) * 1e3 / 3)

    # ---- roofline of the dominant kernel class (the MLP GEMMs)
    counts = P.plan_stats(params, cfg, ds)
    prof = P.profile_update(params, opt, cfg, ds)
    hbm, bf16, bf16_sus, src = _peaks()
    # the MLP passes: tcgen05 GEMMs + reductions, plus the fused output stage
    # (both output layers' forward/backward around the loss head)
    mlp_ms = prof["gemm"] + prof["heads"]
    gemm_tflops = counts["gemm_flops_per_update"] / (mlp_ms / 1e3) / 1e12
    traffic = None
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if tf.exists():
        traffic = json.loads(tf.read_text()).get("tc_gemm_dram_bytes_per_update")
    # Which floor binds the MLP phase: tensor pipe (algorithmic FLOPs at the
    # bf16 peak) or HBM (the DRAM bytes ncu measured for these launches at the
    # measured copy bandwidth)?  The layer-by-layer schedule materialises every
    # activation, so its HBM floor sits above the tensor floor.
    flops = counts["gemm_flops_per_update"]
    tensor_floor_ms = flops / (bf16_sus * 1e12) * 1e3
    hbm_floor_ms = traffic / (hbm * 1e9) * 1e3 if traffic else 0.0
    # per-phase tensor view: the hidden-layer GEMM FLOPs of each phase of the
    # tcgen05 schedule over its measured time (the output layers run in the
    # fused output stage, "heads")
    rows_upd = cfg.epochs * (T * N // world if strong else T * N)
    fwd_mac = dx_mac = 0
    for dims in ((od, *hid), (cd, *hid)):
        for i in range(len(dims) - 1):
            fwd_mac += dims[i] * dims[i + 1]
            if i > 0:
                dx_mac += dims[i] * dims[i + 1]
    phase_fl = {"mlp_forward": 2.0 * fwd_mac * rows_upd, "bwd_dx": 2.0 * dx_mac * rows_upd,
                "bwd_dw": 2.0 * fwd_mac * rows_upd}
    phase_tflops = {k: (phase_fl[k] / (prof[k] / 1e3) / 1e12 if prof.get(k) else None)
                    for k in phase_fl}
    tensor_view = {"achieved": gemm_tflops, "peak": bf16_sus, "unit": "TFLOP/s",
                   "frac": gemm_tflops / bf16_sus, "floor_ms": tensor_floor_ms,
                   "peak_source": f"{src} bf16 sustained (MEASURED_PEAKS.json)",
                   "phase_tflops": phase_tflops,
                   "phase_frac": {k: (v / bf16_sus if v else None) for k, v in phase_tflops.items()}}
    kernel_desc = ("MLP passes of one update: tcgen05 GEMMs (tc_gemm_kernel: grouped forward, "
                   "ELU-gradient dX, one batched dW launch per step) + split-K reductions + the "
                   "fused output stage (ppo_fused_mma_kernel); traffic = ncu DRAM bytes of the "
                   "tc_gemm launches per update (profiles/ncu_traffic.json)")
    if traffic and hbm_floor_ms > tensor_floor_ms:
        gbs = traffic / (mlp_ms / 1e3) / 1e9
        roofline = {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s",
                    "frac": gbs / hbm, "traffic": traffic, "floor_ms": hbm_floor_ms,
                    "tensor": tensor_view, "kernel": kernel_desc,
                    "peak_source": f"{src} HBM copy bandwidth (MEASURED_PEAKS.json)",
                    "algorithmic_flops_per_update": flops, "phase_ms_per_update": prof}
    else:
        roofline = dict(tensor_view, bound="tensor", traffic=traffic, kernel=kernel_desc,
                        algorithmic_flops_per_update=flops, phase_ms_per_update=prof,
                        hbm_floor_ms=hbm_floor_ms)
    # memory-bound kernels at sizes above L2 (tools/bench_kernels.py): GAE /
    # V-trace scans, minibatch / replay gathers, Welford, Polyak, Adam
    hbm_kernels = None
    if rank == 0:
        import importlib.util

        spec = importlib.util.spec_from_file_location("bench_kernels",
                                                      ROOT / "tools" / "bench_kernels.py")
        bk = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(bk)
        hbm_kernels = {k: {"gbs": v["gbs"], "frac": v["frac"]} for k, v in bk.run(hbm).items()}
        hbm_kernels["peak_gbs"] = hbm
        hbm_kernels["note"] = ("algorithmic bytes / CUDA-event time, back-to-back launches, "
                               "inputs larger than L2; frac of the measured copy bandwidth")
        torch.cuda.empty_cache()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": {"fp32": "f32", "tf32": "tf32 (f32 storage/accum)",
                  "bf16": "bf16 GEMM operands/activations, f32 accum/params/optimizer"}[prec],
        "data": "synthetic",
        "config": {"workload": "PPO update (GAE + 5 epochs x 4 minibatches), cfg2 locomotion "
                               "shape: 4096 envs x 24 steps per GPU, obs 235 / act 12, "
                               "actor+critic 512-256-128",
                   "global_batch": transitions, "minibatch_rows": transitions // 4,
                   "parallelism": f"dp{world}", "indices": "device permutation (performance "
                   "mode)", "inputs_larger_than_l2": True,
                   "segment_bytes_per_gpu": ds.h2d_bytes(seg), "gemm_precision": prec_name},
        "update_ms": ms,
        "tf32_arm": tf32,
        "tf32x3_arm": arms.get("tf32x3"),
        "parity_mode": {"value": transitions / (par_ms / 1e3), "unit": UNIT, "update_ms": par_ms,
                        "indices": "host numpy Philox permutation per epoch (reference stream), "
                                   "drawn while the previous epoch runs (one CUDA graph per epoch)",
                        "host_index_gen_ms_per_update": host_perm_ms},
        "e2e": {"value": transitions / (e2e_ms / 1e3), "unit": UNIT,
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "ms_per_step": e2e_ms, "steps": e2e_steps,
                "api": "algos.PpoPipeline.update_async (double-buffered pinned H2D ring, GAE on device, stats read one update behind), "
                       "pinned host segment",
                "serial_gae_ppo_update_ms": serial_ms},
        "roofline": roofline,
        "hbm_kernels": hbm_kernels,
        "clocks": smi.summary(),
        "gpu_launches": int((counts["kernels_per_update"] + 1) * args.steps),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r = cpu_reference_run(2, 1, budget_s=20.0)
        line["cpu_baseline"] = {
            "value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": r["kind"],
            "update_ms": r["update_ms"], "seconds": r["seconds"], "threads_1": r["threads_1"],
            "sample": f"{r['steps_run']} whole cfg2 learner iterations (GAE + ppo_update) of the "
                      + ("unmodified reference (baseline/_ref/unilite)" if r["kind"] == "reference"
                         else "numpy oracle port") + f" on {r['cores']} BLAS threads, after 1 warm-up"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = _args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
