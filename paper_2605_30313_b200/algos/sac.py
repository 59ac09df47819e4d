"""Soft actor-critic on the device (mirror of R:algos/sac.py).

``sac_update`` keeps the reference signature and order (target -> q1 Adam ->
q2 Adam -> [actor + alpha every policy_frequency] -> Polyak) and runs the
native SAC plan (ul_sac_plan_*, csrc/sac.cu).  Noise: a numpy Generator is
consumed exactly like the reference (eps for the target, then eps for the
actor step, each ``standard_normal((B, A))``: "parity mode"); a
:class:`~paper_2605_30313_b200.algos.ppo.DeviceRng` draws both on the device
(Philox4x32-10, "performance mode").  The batch may be a reference-style dict
(host arrays, RowCodec field names) or a :class:`DeviceRows` handle pointing at
device replay rows (the DeviceReplayCache fast path: no decode, no H2D).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from .. import _dev, _dist, _lib
from ..errors import DivergenceError
from ..tensornet.adam import OptState
from ..tensornet.mlp import ModelParams
from .configs import SacConfig
from .ppo import DeviceRng
from .segment import UpdateStats


@dataclass
class ScalarAdam:
    """R:algos/sac.py:35-53 (host copy of the device alpha optimizer)."""

    lr: float
    m: float = 0.0
    v: float = 0.0
    t: int = 0
    betas: tuple = (0.9, 0.999)
    eps: float = 1e-8

    def step(self, x: float, g: float) -> float:
        if not np.isfinite(g):
            raise DivergenceError("non-finite gradient in ScalarAdam")
        self.t += 1
        b1, b2 = self.betas
        self.m = b1 * self.m + (1 - b1) * g
        self.v = b2 * self.v + (1 - b2) * g * g
        m_hat = self.m / (1 - b1 ** self.t)
        v_hat = self.v / (1 - b2 ** self.t)
        return x - self.lr * m_hat / (np.sqrt(v_hat) + self.eps)


@dataclass
class SacParams:
    """R:algos/sac.py:56-69."""

    actor: ModelParams
    q1: ModelParams
    q2: ModelParams
    q1_targ: ModelParams
    q2_targ: ModelParams
    log_alpha: float

    def copy(self) -> "SacParams":
        return SacParams(self.actor.copy(), self.q1.copy(), self.q2.copy(), self.q1_targ.copy(),
                         self.q2_targ.copy(), self.log_alpha)


@dataclass
class SacState:
    """R:algos/sac.py:72-97."""

    params: SacParams
    actor_opt: OptState
    q1_opt: OptState
    q2_opt: OptState
    alpha_opt: ScalarAdam
    action_dim: int
    update_count: int = 0

    @classmethod
    def create(cls, actor: ModelParams, q1: ModelParams, q2: ModelParams,
               cfg: SacConfig) -> "SacState":
        params = SacParams(actor=actor, q1=q1, q2=q2, q1_targ=q1.copy(), q2_targ=q2.copy(),
                           log_alpha=float(np.log(cfg.alpha_init)))
        return cls(params=params, actor_opt=OptState.for_params(actor, cfg.actor_lr),
                   q1_opt=OptState.for_params(q1, cfg.critic_lr),
                   q2_opt=OptState.for_params(q2, cfg.critic_lr),
                   alpha_opt=ScalarAdam(lr=cfg.alpha_lr), action_dim=actor.arch.output_dim)


def soft_update(target: ModelParams, online: ModelParams, tau: float) -> None:
    """target <- (1 - tau) target + tau online, in place (R:algos/sac.py:100-108)."""
    _lib.call("ul_polyak", _dev.ptr(target.buf), _dev.ptr(online.buf), target.buf.numel(),
              float(tau), _dev.stream())


class DeviceRows:
    """A replay batch still in codec-row form on the device: rows of
    ``ring[idx[i] % modulo]`` (pitch in floats).  Produced by
    :class:`~paper_2605_30313_b200.replaypath.DeviceReplayCache`."""

    def __init__(self, ring: torch.Tensor, pitch: int, idx: torch.Tensor | None, n: int,
                 modulo: int = 0, lo: int = 0, hi: int = 2**62):
        self.ring, self.pitch, self.idx, self.n = ring, pitch, idx, n
        self.modulo, self.lo, self.hi = modulo, lo, hi


# ------------------------------------------------------------------- plan
class _SacPlan:
    def __init__(self, state: SacState, batch: int, cfg: SacConfig, world: int = 1):
        d = _lib.SacPlanDesc()
        p = state.params
        d.actor = p.actor.arch.desc()
        d.critic = p.q1.arch.desc()
        d.batch = batch
        d.obs_dim = p.actor.arch.input_dim
        d.act_dim = p.actor.arch.output_dim
        d.gamma, d.tau = cfg.gamma, cfg.tau
        d.target_entropy = -cfg.target_entropy_ratio * state.action_dim
        d.max_grad_norm = cfg.max_grad_norm
        # every SAC GEMM (critics, targets, actor, and the critics' dQ/da input
        # gradient with its fp32 output) runs on the selected back end
        d.gemm_backend = _lib.gemm_backend()
        d.world_size = world
        h = C.c_void_p()
        _lib.call("ul_sac_plan_create", C.byref(d), C.byref(h))
        self.h, self.desc, self.batch, self.world = h, d, batch, world
        # data-parallel all-reduce buffers (torch-owned so torch.distributed
        # can reduce them in place; bound into the plan)
        self.red = None
        if world > 1:
            pq, pa = p.q1.arch.param_count, p.actor.arch.param_count
            dev = p.actor.buf.device
            self.red = (_dev.zeros(2 * pq + 4, torch.float32, dev),
                        _dev.zeros(pa + 4, torch.float32, dev))
        self.n_cap = 0
        self.eps_ptr = None
        self.reserve(1)
        self._bound = None
        self.stage = None

    def reserve(self, n: int) -> None:
        """Noise / statistics room for runs of n updates."""
        if n <= self.n_cap:
            return
        _lib.call("ul_sac_plan_reserve", self.h, int(n))
        eps = C.c_void_p()
        _lib.call("ul_sac_plan_noise_ptr", self.h, C.byref(eps))
        self.eps_ptr, self.n_cap = eps.value, n
        self.stats_h = _dev.pinned_empty((n, 4), np.float64)

    def __del__(self):
        try:
            if self.h:
                _lib.lib().ul_sac_plan_destroy(self.h)
        except Exception:
            pass

    def bind(self, state: SacState):
        p = state.params
        key = (p.actor.buf.data_ptr(), p.q1.buf.data_ptr(), p.q2.buf.data_ptr(),
               p.q1_targ.buf.data_ptr(), p.q2_targ.buf.data_ptr(),
               state.actor_opt.m.buf.data_ptr(), state.q1_opt.m.buf.data_ptr(),
               state.q2_opt.m.buf.data_ptr())
        if key == self._bound:
            return
        b = _lib.SacBindings()
        vals = dict(actor=p.actor.buf, actor_m=state.actor_opt.m.buf,
                    actor_v=state.actor_opt.v.buf, q1=p.q1.buf, q1_m=state.q1_opt.m.buf,
                    q1_v=state.q1_opt.v.buf, q2=p.q2.buf, q2_m=state.q2_opt.m.buf,
                    q2_v=state.q2_opt.v.buf, q1t=p.q1_targ.buf, q2t=p.q2_targ.buf)
        if self.red is not None:
            vals["critic_red"], vals["actor_red"] = self.red
        for k, v in vals.items():
            setattr(b, k, _dev.ptr(v))
        _lib.call("ul_sac_plan_bind", self.h, C.byref(b))
        self._bound = key


_PLANS: dict = {}


def _plan_for(state: SacState, batch: int, cfg: SacConfig, world: int = 1,
              rank: int = 0) -> _SacPlan:
    p = state.params
    key = (p.actor.arch, p.q1.arch, batch, cfg.gamma, cfg.tau, cfg.target_entropy_ratio,
           cfg.max_grad_norm, _lib.gemm_backend(), torch.cuda.current_device(), world, rank)
    plan = _PLANS.get(key)
    if plan is None:
        plan = _SacPlan(state, batch, cfg, world)
        _PLANS[key] = plan
    plan.bind(state)
    return plan


_PINNED: dict = {}


def _pinned(key, shape, dtype=np.float32) -> np.ndarray:
    """Reusable page-locked staging (callers sync before reuse: sac_update
    reads its statistics back at the end of every call)."""
    buf = _PINNED.get(key)
    if buf is None or buf.shape != tuple(shape):
        buf = _dev.pinned_empty(shape, dtype)
        _PINNED[key] = buf
    return buf


def _encode_rows(batch: dict, obs_dim: int, act_dim: int) -> np.ndarray:
    """RowCodec.encode (R:replaypath/storage.py:25-35) into a pinned staging row block."""
    n = len(batch["obs"])
    width = 2 * obs_dim + act_dim + 3
    rows = _pinned(("rows", n, width, _dist.world_info()[1]), (n, width))
    d, a = obs_dim, act_dim
    rows[:, :d] = _dev.to_numpy(batch["obs"])
    rows[:, d:d + a] = _dev.to_numpy(batch["action"])
    rows[:, d + a] = _dev.to_numpy(batch["reward"])
    rows[:, d + a + 1:2 * d + a + 1] = _dev.to_numpy(batch["next_obs"])
    rows[:, 2 * d + a + 1] = np.asarray(_dev.to_numpy(batch["terminated"]), np.float32)
    rows[:, 2 * d + a + 2] = np.asarray(_dev.to_numpy(batch["n_used"]), np.float32)
    return rows


def _load_batch(plan: _SacPlan, batch, obs_dim: int, act_dim: int) -> None:
    s = _dev.stream()
    if isinstance(batch, DeviceRows):
        _lib.call("ul_sac_plan_load_rows", plan.h, _dev.ptr(batch.ring), batch.pitch,
                  _dev.ptr(batch.idx) if batch.idx is not None else None, batch.modulo,
                  batch.lo, batch.hi, None, s)
        return
    rows_dev = getattr(batch, "rows", None)
    if isinstance(rows_dev, torch.Tensor) and rows_dev.is_cuda:
        # DeviceBatch from DeviceReplayCache / RowCodec.decode: rows already in HBM
        _lib.call("ul_sac_plan_load_rows", plan.h, _dev.ptr(rows_dev), rows_dev.stride(0), None,
                  0, 0, 2**62, None, s)
        return
    rows = _encode_rows(batch, obs_dim, act_dim)
    if plan.stage is None or tuple(plan.stage.shape) != rows.shape:
        plan.stage = torch.empty(rows.shape, dtype=torch.float32, device="cuda")
    dev = plan.stage
    _dev.h2d(dev, rows)
    _lib.call("ul_sac_plan_load_rows", plan.h, _dev.ptr(dev), rows.shape[1], None, 0, 0,
              2**62, None, s)


def _fill_noise(plan: _SacPlan, rng, B: int, A: int, actor_steps, world: int = 1,
                rank: int = 0) -> None:
    """Noise for this rank's B rows of len(actor_steps) consecutive updates.
    Host Generator: the reference's global [B*world, A] draws in the
    reference order (per update: the target's eps, then the actor step's
    when it runs), this rank's row slice; device RNG: the rank folded into
    the stream key."""
    s = _dev.stream()
    n = len(actor_steps)
    plan.reserve(n)
    if rng is None or isinstance(rng, DeviceRng):
        rng = rng if rng is not None else DeviceRng(0)
        key = rng.next_key() ^ (0x9E3779B97F4A7C15 * rank & 0xFFFFFFFFFFFFFFFF)
        _lib.call("ul_sac_plan_device_noise", plan.h, key, rng.counter, s)
        return
    eps = _pinned(("eps", B, A, rank, n), (n, 2, B, A))
    lo, hi = rank * B, (rank + 1) * B
    for u, do_actor in enumerate(actor_steps):
        eps[u, 0] = rng.standard_normal((B * world, A))[lo:hi]      # critic_target (R:algos/sac.py:117)
        if do_actor:
            eps[u, 1] = rng.standard_normal((B * world, A))[lo:hi]  # actor step (R:algos/sac.py:237)
    _lib.call("ul_memcpy_async", plan.eps_ptr, eps.ctypes.data, eps.nbytes, s)


def _shard_batch(batch, world: int, rank: int):
    """This rank's contiguous 1/world slice of a global batch (SURVEY.md 8(e):
    the host draws the global indices, each rank gathers its rows)."""
    if world == 1:
        return batch
    if isinstance(batch, DeviceRows):
        if batch.n % world:
            raise ValueError("world_size must divide the SAC batch")
        per = batch.n // world
        idx = batch.idx[rank * per:(rank + 1) * per] if batch.idx is not None else None
        if idx is None:
            raise ValueError("data-parallel SAC needs an index vector for DeviceRows batches")
        return DeviceRows(batch.ring, batch.pitch, idx, per, batch.modulo, batch.lo, batch.hi)
    n = len(batch["obs"])
    if n % world:
        raise ValueError("world_size must divide the SAC batch")
    per = n // world
    return {k: v[rank * per:(rank + 1) * per] for k, v in batch.items()}


def sac_update(batch, state: SacState, cfg: SacConfig, rng) -> UpdateStats:
    """One critic update (+ periodic actor/alpha update) on a replay batch
    (R:algos/sac.py:139-178)."""
    return sac_updates(batch, state, cfg, rng, 1)[0]


def sac_updates(batch, state: SacState, cfg: SacConfig, rng, n: int) -> list:
    """n consecutive ``sac_update`` calls on one batch -- the learner tick's
    ``updates_per_step`` loop (R:runtime/sac_runner.py:313-321) -- as ONE
    CUDA-graph launch on a single GPU: one control upload, no host round trip
    between updates, one read-back.  Returns the n UpdateStats; raises
    DivergenceError (after updating the host mirrors of the state that did
    advance) at the first update the reference would have raised in."""
    if n < 1:
        raise ValueError("n must be >= 1")
    nrows = batch.n if isinstance(batch, DeviceRows) else len(batch["obs"])
    if nrows < 2:
        raise ValueError("sac_update needs a batch of at least 2 rows")
    world, rank = _dist.world_info()
    batch = _shard_batch(batch, world, rank)
    nrows //= world
    p = state.params
    od, ad = p.actor.arch.input_dim, p.actor.arch.output_dim
    plan = _plan_for(state, nrows, cfg, world, rank)
    _load_batch(plan, batch, od, ad)
    pf = cfg.policy_frequency
    steps = [(state.update_count + u + 1) % pf == 0 for u in range(n)]
    _fill_noise(plan, rng, nrows, ad, steps, world, rank)
    ctl = _lib.SacCtl()
    ctl.log_alpha = p.log_alpha
    ctl.a_m, ctl.a_v, ctl.a_t = state.alpha_opt.m, state.alpha_opt.v, float(state.alpha_opt.t)
    ctl.alpha_lr = state.alpha_opt.lr
    lrs = (C.c_double * 3)(state.actor_opt.lr, state.q1_opt.lr, state.q2_opt.lr)
    ts = (C.c_int64 * 3)(state.actor_opt.t, state.q1_opt.t, state.q2_opt.t)
    s = _dev.stream()
    _lib.call("ul_sac_plan_begin", plan.h, C.byref(ctl), lrs, ts, s)
    alpha0 = float(np.exp(p.log_alpha))
    if world == 1:
        _lib.call("ul_sac_plan_run", plan.h, n, state.update_count, pf, s)
        out = _lib.SacCtl()
        st = _lib.lib().ul_sac_plan_finish(plan.h, C.byref(out), ts, plan.stats_h.ctypes.data,
                                          n, s)
        rows = plan.stats_h[:n].copy()
    else:
        if n != 1:
            raise ValueError("data-parallel SAC runs one update per call")
        # the two exchange points of SURVEY.md 8(e): critic grads (+ loss), then
        # actor grads (+ loss, sum log pi) on actor steps; Polyak stays local
        _lib.call("ul_sac_plan_critic_grads", plan.h, s)
        _dist.all_reduce_sum(plan.red[0])
        _lib.call("ul_sac_plan_critic_apply", plan.h, s)
        if steps[0]:
            _lib.call("ul_sac_plan_actor_grads", plan.h, s)
            _dist.all_reduce_sum(plan.red[1])
            _lib.call("ul_sac_plan_actor_apply", plan.h, s)
        _lib.call("ul_sac_plan_polyak", plan.h, s)
        out = _lib.SacCtl()
        st = _lib.lib().ul_sac_plan_finish(plan.h, C.byref(out), ts, None, 0, s)
        rows = np.array([[out.critic_loss, out.actor_loss if steps[0] else np.nan,
                          out.alpha_loss if steps[0] else np.nan,
                          float(np.exp(out.log_alpha)) if steps[0] else alpha0]])
    state.actor_opt.t, state.q1_opt.t, state.q2_opt.t = int(ts[0]), int(ts[1]), int(ts[2])
    # updates that completed (the reference counts an update once its critic
    # step is finite, R:algos/sac.py:158-163; an actor-side failure comes after)
    fail = int(out.fail_update) if st != 0 else n
    counted = fail + (1 if st != 0 and out.diverged == 2 else 0)
    state.update_count += counted
    p.log_alpha = float(out.log_alpha)
    state.alpha_opt.m, state.alpha_opt.v = float(out.a_m), float(out.a_v)
    state.alpha_opt.t = int(round(out.a_t))
    if st != 0:
        _lib.check(st, "ul_sac_plan_finish")
    stats = []
    for u in range(n):
        su = UpdateStats(lr=cfg.critic_lr)
        su.extra["critic_loss"] = float(rows[u, 0])
        su.extra["alpha"] = float(rows[u, 3])
        if steps[u]:
            su.extra["actor_loss"] = float(rows[u, 1])
            su.extra["alpha_loss"] = float(rows[u, 2])
        stats.append(su)
    return stats


# ------------------------------------------------- per-call drop-in API
# The reference's building blocks of sac_update (R:algos/__init__.py:24-27),
# each on the device: network passes through tensornet (tcgen05 / SIMT
# kernels), the heads through ul_sac_* kernels (csrc/sac_api.cu).
def _concat_cols(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """[a | b] rows on the device (one gather launch, no host round trip)."""
    n, da = a.shape
    db = b.shape[1]
    out = torch.empty((n, _dev.round_up(da + db, 4)), dtype=torch.float32, device=a.device)
    rb = out.stride(0) * 4
    base = _dev.ptr(out)
    _lib.call("ul_gather_rows", 2, _lib.ptr_array([_dev.ptr(a), _dev.ptr(b)]),
              _lib.ptr_array([base, base + 4 * da]),
              _lib.i64_array([a.stride(0) * 4, b.stride(0) * 4]), _lib.i64_array([rb, rb]),
              _lib.i64_array([4 * da, 4 * db]), None, None, n, 0, 0, 2**62, None, _dev.stream())
    return out[:, :da + db]


def critic_target(params: SacParams, batch: dict, gamma: float, rng) -> torch.Tensor:
    """y for both critics, no gradients (R:algos/sac.py:111-125); float64
    [B] on the device.  eps is the reference's standard_normal draw."""
    from ..tensornet.distributions import sample_squashed
    from ..tensornet.mlp import forward, value_forward

    nxt = _dev.to_device_f32(batch["next_obs"])
    mean, _ = forward(params.actor, nxt)
    n, A = mean.shape
    eps = rng.standard_normal((n, A))
    a, _, logp = sample_squashed(mean, params.actor.log_std, eps)
    qin = _concat_cols(nxt, a)
    q1t, _ = value_forward(params.q1_targ, qin)
    q2t, _ = value_forward(params.q2_targ, qin)
    r = _dev.to_device_f64(batch["reward"])
    term = _dev.to_device_f64(np.asarray(_dev.to_numpy(batch["terminated"]), np.float64))
    nu = _dev.to_device_f64(batch["n_used"])
    y = torch.empty(n, dtype=torch.float64, device=mean.device)
    q1c, q2c = q1t.contiguous(), q2t.contiguous()
    _lib.call("ul_sac_soft_target", _dev.ptr(r), _dev.ptr(term), _dev.ptr(nu), _dev.ptr(q1c),
              _dev.ptr(q2c), _dev.ptr(logp), float(params.log_alpha), float(gamma), n,
              _dev.ptr(y), _dev.stream())
    return y


def critic_loss_and_grads(q_params: ModelParams, q_in, y):
    """MSE of one critic against a fixed target, exact gradients
    (R:algos/sac.py:128-136): (loss, grads, q_pred)."""
    from ..tensornet.mlp import backward, value_forward

    q_pred, cache = value_forward(q_params, q_in)
    n = q_pred.shape[0]
    yd = _dev.to_device_f64(y)
    qc = q_pred.contiguous()
    dq = torch.empty((n, 1), dtype=torch.float32, device=qc.device)
    loss = torch.empty(1, dtype=torch.float64, device=qc.device)
    _lib.call("ul_sac_mse_head", _dev.ptr(qc), _dev.ptr(yd), n, _dev.ptr(dq), _dev.ptr(loss),
              _dev.ptr(_dev.api_work()), _dev.stream())
    _, grads = backward(q_params, cache, dq)
    return float(loss.item()), grads, q_pred


def actor_loss_and_grads(params: SacParams, obs, eps):
    """Reparameterized actor loss mean(alpha logpi - min Q) with exact grads
    (R:algos/sac.py:181-221): (loss, actor grads, logp)."""
    from ..tensornet.distributions import sample_squashed
    from ..tensornet.mlp import backward, forward, value_forward

    od = _dev.to_device_f32(obs)
    mean, a_cache = forward(params.actor, od)
    n, A = mean.shape
    ed = _dev.to_device_f32(eps)
    a, _, logp = sample_squashed(mean, params.actor.log_std, ed)
    qin = _concat_cols(od, a)
    q1p, c1 = value_forward(params.q1, qin)
    q2p, c2 = value_forward(params.q2, qin)
    d1 = torch.empty((n, 1), dtype=torch.float32, device=mean.device)
    d2 = torch.empty_like(d1)
    loss = torch.empty(1, dtype=torch.float64, device=mean.device)
    work = _dev.api_work()
    q1c, q2c = q1p.contiguous(), q2p.contiguous()
    _lib.call("ul_sac_pick_head", _dev.ptr(q1c), _dev.ptr(q2c), _dev.ptr(logp), n,
              float(params.log_alpha), _dev.ptr(d1), _dev.ptr(d2), _dev.ptr(loss),
              _dev.ptr(work), _dev.stream())
    din1, _ = backward(params.q1, c1, d1)
    din2, _ = backward(params.q2, c2, d2)
    D = od.shape[1]
    dmean = torch.empty((n, A), dtype=torch.float32, device=mean.device)
    dls = _dev.zeros(A, torch.float32, mean.device)
    ls = params.actor.log_std.contiguous()
    edc = ed.contiguous()
    _lib.call("ul_sac_actor_head", _dev.ptr(a), _dev.ptr(edc), _dev.ptr(din1[:, D:]),
              _dev.ptr(din2[:, D:]), din1.stride(0), _dev.ptr(ls), n, A,
              float(params.log_alpha), _dev.ptr(dmean), _dev.ptr(dls), _dev.ptr(work),
              _dev.stream())
    _, grads = backward(params.actor, a_cache, dmean)
    off = grads.buf.numel() - A
    _lib.call("ul_memcpy_async", _dev.ptr(grads.buf) + 4 * off, _dev.ptr(dls), 4 * A,
              _dev.stream())  # (backward leaves the actor's log_std gradient at zero)
    return float(loss.item()), grads, logp


def alpha_loss_and_grad(log_alpha: float, logp, target_entropy: float) -> tuple:
    """Temperature loss -log_alpha * mean(logpi + H) and its gradient
    (R:algos/sac.py:224-229); logpi is a constant."""
    lp = _dev.to_device_f32(logp).reshape(-1).contiguous()
    out = torch.empty(1, dtype=torch.float64, device=lp.device)
    _lib.call("ul_sum_f64", _dev.ptr(lp), lp.numel(), float(target_entropy), _dev.ptr(out),
              _dev.ptr(_dev.api_work()), _dev.stream())
    excess = float(out.item()) / lp.numel()
    return -log_alpha * excess, -excess
