"""Clipped-surrogate PPO on the device (mirror of R:algos/ppo.py).

``ppo_update`` keeps the reference signature.  It stages the segment into HBM,
draws the per-epoch minibatch permutations exactly as the reference does
(``rng.permutation(n)`` per epoch, R:algos/ppo.py:162) when ``rng`` is a numpy
Generator ("parity mode"), or on the device when ``rng`` is a
:class:`DeviceRng` ("performance mode"), and replays the native update plan
(ul_ppo_plan_*) -- a single CUDA graph per update on one GPU.  Under
torch.distributed with world_size > 1 each rank takes its 1/G slice of every
minibatch and the plan's gradient buffer is all-reduced (NCCL) between the
backward and the optimizer step.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from .. import _dev, _dist, _lib
from ..errors import DivergenceError
from ..tensornet.adam import OptState
from ..tensornet.mlp import Grads, ModelParams
from ._staging import staging_for
from .configs import PpoConfig
from .segment import UpdateStats


@dataclass
class AcParams:
    """R:algos/ppo.py:38-46."""

    actor: ModelParams
    critic: ModelParams

    def copy(self) -> "AcParams":
        return AcParams(self.actor.copy(), self.critic.copy())


@dataclass
class AcOpt:
    """R:algos/ppo.py:49-67."""

    actor: OptState
    critic: OptState

    @classmethod
    def for_params(cls, params: AcParams, lr: float) -> "AcOpt":
        return cls(OptState.for_params(params.actor, lr), OptState.for_params(params.critic, lr))

    @property
    def lr(self) -> float:
        return self.actor.lr

    def set_lr(self, lr: float) -> None:
        self.actor.lr = lr
        self.critic.lr = lr


class DeviceRng:
    """Performance-mode minibatch index source: a keyed device permutation per
    epoch (ul_device_permutation).  Statistically a uniform shuffle, NOT the
    numpy Philox stream -- results then match the reference in distribution,
    not bit-for-bit."""

    def __init__(self, seed: int = 0):
        self.seed = int(seed)
        self.counter = 0

    def next_key(self) -> int:
        self.counter += 1
        x = (self.seed * 0x9E3779B97F4A7C15 + self.counter * 0xBF58476D1CE4E5B9) & (2**64 - 1)
        x ^= x >> 31
        return x


# ------------------------------------------------------------------- plans
class _Plan:
    def __init__(self, desc: _lib.PpoPlanDesc):
        h = C.c_void_p()
        _lib.call("ul_ppo_plan_create", C.byref(desc), C.byref(h))
        self.h = h
        self.desc = desc
        self._bind_key = None
        self.pending = None  # unread PendingUpdate whose records this plan holds
        n = C.c_int64()
        p = C.c_void_p()
        _lib.call("ul_ppo_plan_reduce_buffer", self.h, C.byref(p), C.byref(n))
        self.red_len = n.value

    def __del__(self):
        try:
            if self.h:
                _lib.lib().ul_ppo_plan_destroy(self.h)
        except Exception:
            pass

    def bind(self, ds, adv, ret, oldv, params: AcParams, opt: AcOpt, red=None):
        b = _lib.PpoBindings()
        vals = dict(obs=ds.obs, cobs=ds.cobs, act=ds.act, blogp=ds.blogp, adv=adv, ret=ret,
                    oldv=oldv, actor_params=params.actor.buf, critic_params=params.critic.buf,
                    actor_m=opt.actor.m.buf, actor_v=opt.actor.v.buf, critic_m=opt.critic.m.buf,
                    critic_v=opt.critic.v.buf, perm=ds.perm, reduce_buf=red)
        ptrs = tuple(_dev.ptr(v) if v is not None else None for v in vals.values())
        if ptrs == self._bind_key:  # same buffers: the bound plan (and its graph) stands
            return
        for k, v in zip(vals, ptrs):
            setattr(b, k, v)
        _lib.call("ul_ppo_plan_bind", self.h, C.byref(b))
        self._bind_key = ptrs


_PLANS: dict = {}


def release_slots(prefix: str) -> None:
    """Drop the staging segments and update plans of every slot whose name
    starts with `prefix` (a PpoPipeline's own slots)."""
    from . import _staging

    for k in [k for k in _PLANS if str(k[-1]).startswith(prefix)]:
        del _PLANS[k]
    for k in [k for k in _staging._CACHE if str(k[0]).startswith(prefix)]:
        del _staging._CACHE[k]


def _plan_for(params: AcParams, cfg: PpoConfig, ds, world: int, rank: int,
              raw_adv: bool = False) -> _Plan:
    # one plan (and CUDA graph) per staging slot: the pipeline alternates two
    key = (params.actor.arch, params.critic.arch, ds.rows, ds.ld, cfg.epochs, cfg.minibatches,
           cfg.clip_param, cfg.entropy_coef, cfg.value_loss_coef, cfg.use_clipped_value_loss,
           cfg.max_grad_norm, world, rank, raw_adv, _dist.segment_mode(), _dist.dp_forced(),
           _lib.gemm_backend(), torch.cuda.current_device(), getattr(ds, "slot", "ppo"),
           getattr(ds, "bf16_rows", False))
    plan = _PLANS.get(key)
    if plan is None:
        d = _lib.PpoPlanDesc()
        d.actor = params.actor.arch.desc()
        d.critic = params.critic.arch.desc()
        d.rows = ds.rows
        d.ld_obs, d.ld_cobs, d.ld_act = ds.ld
        d.epochs, d.minibatches = cfg.epochs, cfg.minibatches
        d.clip_param, d.entropy_coef = cfg.clip_param, cfg.entropy_coef
        d.value_loss_coef = cfg.value_loss_coef
        d.use_clipped_value_loss = int(cfg.use_clipped_value_loss)
        d.max_grad_norm = cfg.max_grad_norm
        d.world_size, d.rank, d.raw_advantages = world, rank, int(raw_adv)
        d.local_shards = int(_dist.segment_mode() == "local" and _dp_path(world))
        d.gemm_backend = _lib.gemm_backend()
        d.obs_bf16 = int(getattr(ds, "bf16_rows", False))
        plan = _Plan(d)
        _PLANS[key] = plan
    return plan


_PINNED_PERM: dict = {}


def fill_permutations(ds, rng, epochs: int) -> None:
    """Per-epoch permutations into ds.perm: host Philox (parity) or device."""
    n = ds.rows
    if rng is None or isinstance(rng, DeviceRng):
        rng = rng if rng is not None else DeviceRng(0)
        keys = (C.c_uint64 * epochs)(*[rng.next_key() for _ in range(epochs)])
        _lib.call("ul_device_permutations", n, epochs, keys, _dev.ptr(ds.perm), ds.perm.stride(0),
                  _dev.stream())
        return
    key = (n, epochs, _dist.world_info()[1])
    host = _PINNED_PERM.get(key)
    if host is None:
        host = _dev.pinned_empty((epochs, n), np.int64)
        _PINNED_PERM[key] = host
    # the pinned buffer may still be read by a previous async copy
    _lib.call("ul_stream_sync", _dev.stream())
    for e in range(epochs):
        host[e] = rng.permutation(n)
    _dev.h2d(ds.perm[:epochs], host)


def _world():
    return _dist.world_info()


class PendingUpdate:
    """An update enqueued behind earlier ones without a host round trip
    (``PpoPipeline.update_async``).  ``result()`` waits for this update's
    result records only -- later updates may already be queued behind it --
    and returns its ``UpdateStats``; results are read in launch order."""

    def __init__(self, plan: _Plan, opt: AcOpt):
        self.plan, self.opt = plan, opt
        self._stats = None
        self._err = None
        self.t_after = None  # (actor t, critic t) the device reported

    @property
    def done(self) -> bool:
        return self._stats is not None or self._err is not None

    def _finish(self) -> None:
        if self.done:
            return
        try:
            self._stats = _stats(finish_plan(self.plan, self.opt), self.opt)
        except Exception as e:  # (DivergenceError: raised by result())
            self._err = e
        self.t_after = (self.opt.actor.t, self.opt.critic.t)
        if self.plan.pending is self:
            self.plan.pending = None

    def result(self) -> UpdateStats:
        if not self.done:
            _drain_pending(upto=self)
        if self._err is not None:
            raise self._err
        return self._stats


_PENDING: list = []  # enqueued, unread chained updates in launch order


def _drain_pending(upto=None) -> None:
    """Read pending chained updates in launch order (through `upto`, else all),
    so the host copy of the Adam step counters is current again."""
    if upto is not None and upto not in _PENDING:
        upto._finish()  # (not queued: nothing older to read first)
        return
    while _PENDING:
        h = _PENDING.pop(0)
        h._finish()
        if h is upto:
            break


def launch_plan(plan: _Plan, params: AcParams, opt: AcOpt, world: int, red,
                prev: _Plan | None = None) -> None:
    """Enqueue one update (single GPU: one CUDA-graph launch, no host wait).
    prev: the plan of the update this one is chained behind on the device
    (its step counters / divergence latch continue from prev's controller).
    Data-parallel (world > 1): the controller upload + advantage statistics
    (all-reduced across "local" shards), then the 20 x (step_grads -> NCCL
    all-reduce of the gradient buffer -> step_apply) sequence -- captured once
    per bound plan as ONE CUDA graph with the NCCL all-reduces inside it."""
    s = _dev.stream()
    cfgd = plan.desc
    if not _dp_path(world) and prev is not None:
        _lib.call("ul_ppo_plan_run_after", plan.h, prev.h, opt.actor.lr, opt.critic.lr, s)
        return
    if not _dp_path(world):
        _lib.call("ul_ppo_plan_run", plan.h, opt.actor.lr, opt.critic.lr, opt.actor.t,
                  opt.critic.t, 1, s)
        return
    def prologue():
        _lib.call("ul_ppo_plan_begin", plan.h, opt.actor.lr, opt.critic.lr, opt.actor.t,
                  opt.critic.t, s)
        if cfgd.local_shards and not cfgd.raw_advantages:
            sums = _dist.sums_buffer(3)
            _lib.call("ul_ppo_plan_adv_sums", plan.h, _dev.ptr(sums), s)
            _dist.all_reduce_sum(sums)
            _lib.call("ul_ppo_plan_adv_finalize", plan.h, _dev.ptr(sums), s)

    prologue()

    def steps():
        st = _dev.stream()
        for e in range(cfgd.epochs):
            for k in range(cfgd.minibatches):
                _lib.call("ul_ppo_plan_step_grads", plan.h, e, k, st)
                _dist.all_reduce_sum(red)
                _lib.call("ul_ppo_plan_step_apply", plan.h, e, k, st)

    if not _dist.dp_graph_enabled():
        steps()
        return
    key = (plan._bind_key, _dev.ptr(red))
    if getattr(plan, "dp_graph_key", None) != key:
        # capture once per binding (the first update runs eagerly so NCCL's
        # communicator and the plan's lazily built state exist before capture)
        if getattr(plan, "dp_warm", None) != key:
            plan.dp_warm = key
            steps()
            return
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        cs.wait_stream(torch.cuda.current_stream())
        torch.cuda.synchronize()
        try:
            with torch.cuda.graph(g, stream=cs):
                steps()
        except RuntimeError as exc:  # the collective refused capture: stay eager
            _dist.disable_dp_graph(f"{type(exc).__name__}: {exc}")
            torch.cuda.synchronize()
            prologue()  # (nothing captured ran: restart the update eagerly)
            steps()
            return
        plan.dp_graph, plan.dp_graph_key = g, key
    plan.dp_graph.replay()


def _dp_path(world: int) -> bool:
    return world > 1 or _dist.dp_forced()


def finish_plan(plan: _Plan, opt: AcOpt) -> _lib.PpoResult:
    """Read the update's statistics (the step's device->host result)."""
    res = _lib.PpoResult()
    st = _lib.lib().ul_ppo_plan_finish(plan.h, C.byref(res), _dev.stream())
    opt.actor.t = int(res.t_actor)
    opt.critic.t = int(res.t_critic)
    if st != 0:
        _lib.check(st, "ul_ppo_plan_finish")
    return res


def run_plan(plan: _Plan, params: AcParams, opt: AcOpt, world: int, red) -> _lib.PpoResult:
    launch_plan(plan, params, opt, world, red)
    return finish_plan(plan, opt)


def _launch_epochs(ds, adv, ret, oldv, params, opt, cfg, rng, raw_adv=False, prev=None):
    world, rank = _world()
    plan = _plan_for(params, cfg, ds, world, rank, raw_adv)
    host_rng = rng is not None and not isinstance(rng, DeviceRng)
    if prev is None or _dp_path(world) or host_rng:
        _drain_pending()  # the launch reads the host step counters
        prev = None
    elif plan.pending is not None:
        _drain_pending(upto=plan.pending)  # its result records are about to be reused
    if not _dp_path(world) and host_rng:
        # parity mode: one graph per epoch, so the host draws the reference
        # stream's permutation for epoch e + 1 while epoch e runs
        plan.bind(ds, adv, ret, oldv, params, opt, None)
        _pipelined_host_epochs(plan, ds, rng, cfg.epochs, opt)
        return plan
    fill_permutations(ds, rng, cfg.epochs)
    red = None
    if _dp_path(world):
        red = _dist.reduce_buffer(plan.red_len)
    plan.bind(ds, adv, ret, oldv, params, opt, red)
    launch_plan(plan, params, opt, world, red, prev)
    return plan


def _pipelined_host_epochs(plan, ds, rng, epochs: int, opt) -> None:
    n = ds.rows
    key = (n, epochs, _dist.world_info()[1])
    host = _PINNED_PERM.get(key)
    if host is None:
        host = _dev.pinned_empty((epochs, n), np.int64)
        _PINNED_PERM[key] = host
    s = _dev.stream()
    _lib.call("ul_stream_sync", s)  # the previous update's copies out of `host` are done
    for e in range(epochs):
        host[e] = rng.permutation(n)  # (numpy releases the GIL; the GPU runs epoch e - 1)
        _dev.h2d(ds.perm[e], host[e])
        _lib.call("ul_ppo_plan_run_epoch", plan.h, e, opt.actor.lr, opt.critic.lr, opt.actor.t,
                  opt.critic.t, s)


def _stats(res, opt) -> UpdateStats:
    return UpdateStats(policy_loss=res.policy_loss, value_loss=res.value_loss,
                       entropy=res.entropy, kl=res.kl, lr=opt.lr, grad_norm=res.grad_norm)


def _epochs_on_device(ds, adv, ret, oldv, params, opt, cfg, rng, raw_adv=False) -> UpdateStats:
    plan = _launch_epochs(ds, adv, ret, oldv, params, opt, cfg, rng, raw_adv)
    return _stats(finish_plan(plan, opt), opt)


def _check_dims(segment, params: AcParams):
    od, cd = params.actor.arch.input_dim, params.critic.arch.input_dim
    ad = params.actor.arch.output_dim
    if tuple(segment.obs.shape[2:]) != (od,) or tuple(segment.critic_obs.shape[2:]) != (cd,) \
            or tuple(segment.actions.shape[2:]) != (ad,):
        raise ValueError("segment feature widths do not match the networks")
    return od, cd, ad


def ppo_update(segment, params: AcParams, opt: AcOpt, cfg: PpoConfig, rng) -> UpdateStats:
    """Epochs x minibatches of clipped-surrogate updates on one segment
    (R:algos/ppo.py:202-229).  The segment must carry advantages/returns."""
    if segment.advantages is None or segment.returns is None:
        raise ValueError("segment advantages/returns not computed")
    od, cd, ad = _check_dims(segment, params)
    T, N = segment.horizon, segment.n_envs
    if (T * N) % cfg.minibatches != 0:
        raise ValueError(f"minibatches {cfg.minibatches} must divide batch size {T * N}")
    world, rank = _world()
    ds = staging_for(T, N, od, cd, ad, cfg.epochs, slot="ppo" if world == 1 else f"ppo_r{rank}")
    ds.load(segment)
    return _epochs_on_device(ds, ds.adv, ds.ret, ds.values, params, opt, cfg, rng)


def normalize_advantages(advantages):
    """(A - mean)/(std + 1e-8) (R:algos/ppo.py:132-133).  Host helper for the
    API surface; the update plan folds this into its loss head on device."""
    a = _dev.to_numpy(advantages).astype(np.float64)
    return (a - a.mean()) / (a.std() + 1e-8)


def ppo_loss_and_grads(params: AcParams, obs, critic_obs, actions, behavior_logp, advantages,
                       returns, old_values, cfg: PpoConfig):
    """Loss terms + exact actor/critic gradients of one minibatch, no optimizer
    step (R:algos/ppo.py:70-129).  Runs the plan's grad phase over all rows."""
    from .segment import RolloutSegment

    obs = np.asarray(_dev.to_numpy(obs))
    n = obs.shape[0]

    def one(x):  # (n, ...) -> (1, n, ...): a one-step "segment"
        a = np.asarray(_dev.to_numpy(x))
        return a.reshape(1, n, *a.shape[1:])

    seg = RolloutSegment(obs=one(obs), critic_obs=one(critic_obs), actions=one(actions),
                         behavior_log_prob=one(behavior_logp), rewards=np.zeros((1, n)),
                         terminated=np.zeros((1, n), bool), truncated=np.zeros((1, n), bool),
                         values=one(old_values), bootstrap_value=np.zeros(n),
                         advantages=one(advantages), returns=one(returns))
    od, cd, ad = _check_dims(seg, params)
    cfg1 = PpoConfig(**{**cfg.__dict__, "epochs": 1, "minibatches": 1})
    ds = staging_for(1, n, od, cd, ad, 1, slot="loss")
    ds.load(seg)
    _dev.h2d(ds.perm[0], np.arange(n, dtype=np.int64))
    plan = _plan_for(params, cfg1, ds, 1, 0, raw_adv=True)
    scratch = AcOpt.for_params(params, 0.0)
    plan.bind(ds, ds.adv, ds.ret, ds.values, params, scratch)
    s = _dev.stream()
    _lib.call("ul_ppo_plan_begin", plan.h, 0.0, 0.0, 0, 0, s)
    _lib.call("ul_ppo_plan_step_grads", plan.h, 0, 0, s)
    p = C.c_void_p()
    m = C.c_int64()
    _lib.call("ul_ppo_plan_reduce_buffer", plan.h, C.byref(p), C.byref(m))
    host = np.empty(m.value, np.float32)
    _lib.call("ul_memcpy_async", host.ctypes.data, p.value, host.nbytes, s)
    _lib.call("ul_stream_sync", s)
    pa, pc = params.actor.buf.numel(), params.critic.buf.numel()
    ga = Grads(torch.empty_like(params.actor.buf), params.actor.arch)
    gc = Grads(torch.empty_like(params.critic.buf), params.critic.arch)
    _dev.h2d(ga.buf, host[:pa])
    _dev.h2d(gc.buf, host[pa:pa + pc])
    pol_sum, val_sum, kl_sum = (float(x) for x in host[pa + pc:pa + pc + 3])
    log_std = _dev.to_numpy(params.actor.log_std).astype(np.float64)
    entropy = float(np.sum(log_std + 0.5 * (np.log(2 * np.pi) + 1.0)))
    policy_loss, value_loss = -pol_sum / n, val_sum / n
    total = policy_loss + cfg.value_loss_coef * value_loss - cfg.entropy_coef * entropy
    terms = dict(policy_loss=policy_loss, value_loss=value_loss, entropy=entropy, total=total,
                 kl=kl_sum / n)
    return terms, ga, gc


def adaptive_lr_step(lr: float, measured_kl: float, cfg: PpoConfig, update_index: int) -> float:
    """Dead-band adaptive LR (R:algos/ppo.py:232-250); host scalar logic."""
    if cfg.schedule != "adaptive":
        return lr
    if update_index % cfg.adaptive_lr_update_interval != 0:
        return lr
    if measured_kl > cfg.desired_kl / cfg.adaptive_kl_beta:
        lr = lr / cfg.adaptive_lr_decay
    elif measured_kl < cfg.desired_kl * cfg.adaptive_kl_beta:
        lr = lr * cfg.adaptive_lr_growth
    return float(np.clip(lr, 1e-6, 1e-2))


def gae_into(ds, gamma: float, lam: float) -> None:
    """GAE (K1) over a staged DeviceSegment, writing ds.adv / ds.ret in place."""
    _lib.call("ul_gae_f32", _dev.ptr(ds.rewards), _dev.ptr(ds.values), _dev.ptr(ds.term),
              _dev.ptr(ds.trunc), _dev.ptr(ds.tv) if ds.has_tv else None, _dev.ptr(ds.boot),
              ds.T, ds.N, float(gamma), float(lam), _dev.ptr(ds.adv), _dev.ptr(ds.ret),
              _dev.stream())


def ppo_update_resident(ds, params: AcParams, opt: AcOpt, cfg: PpoConfig, rng) -> UpdateStats:
    """gae + ppo_update on a segment that is already resident in HBM (the
    learner half of R:runtime/ppo_runner.py:95-102 without the H2D)."""
    gae_into(ds, cfg.gamma, cfg.lam)
    return _epochs_on_device(ds, ds.adv, ds.ret, ds.values, params, opt, cfg, rng)


class PpoPipeline:
    """The collector-to-learner transfer path of the north star: a
    double-buffered pinned-host -> HBM staging ring.  Segment i+1 is copied
    (and re-pitched) on a side stream into the idle slot while the update on
    segment i runs; each slot owns its own bound update plan / CUDA graph.
    GAE runs on the device (K1) inside the update, so only the raw rollout
    fields cross PCIe.  Equivalent to ``gae`` + ``ppo_update`` per segment
    (R:runtime/ppo_runner.py:95-102), pipelined.

        pipe = PpoPipeline(params, opt, cfg, rng)
        pipe.prefetch(seg0)
        for it in range(iterations):
            stats = pipe.update(next_segment=seg_next_or_None)
    """

    _ids = iter(range(1 << 62))

    def __init__(self, params: AcParams, opt: AcOpt, cfg: PpoConfig, rng):
        self.params, self.opt, self.cfg, self.rng = params, opt, cfg, rng
        # staging slots (and the plans / CUDA graphs bound to them) are owned
        # by this pipeline alone: two pipelines never share buffers
        self._tag = f"pipe{next(PpoPipeline._ids)}"
        self.copy = torch.cuda.Stream()
        self.ready = [torch.cuda.Event(), torch.cuda.Event()]
        self.free = [torch.cuda.Event(), torch.cuda.Event()]
        self.slots: list = [None, None]
        self.queue: list = []  # slots holding staged, not yet consumed segments
        self.next_slot = 0
        self._prev = None  # plan of the last update (device-chained launches)
        self._last = None  # PendingUpdate of the last chained update

    def close(self) -> None:
        """Release this pipeline's staging slots and plans."""
        _drain_pending()
        release_slots(self._tag)
        self.slots = [None, None]
        self.queue.clear()
        self._prev = self._last = None

    def __del__(self):
        try:
            release_slots(self._tag)
        except Exception:
            pass

    def _chain_ok(self) -> bool:
        """Chain the next update behind the last one on the device only while
        the device-held Adam step counters / divergence latch are the truth:
        not after an update that raised, nor when the host changed the step
        counters since that update was read."""
        h = self._last
        if self._prev is None or h is None:
            return False
        if not h.done:
            return True  # still in flight: the host holds no newer state
        if h._err is not None:
            return False
        return (self.opt.actor.t, self.opt.critic.t) == h.t_after
    def prefetch(self, segment) -> None:
        """Start the H2D of a segment into the idle slot (returns at once when
        the host arrays are pinned)."""
        if len(self.queue) >= 2:
            raise RuntimeError("both staging slots hold segments not yet consumed")
        od, cd, ad = _check_dims(segment, self.params)
        T, N = segment.horizon, segment.n_envs
        if (T * N) % self.cfg.minibatches != 0:
            raise ValueError(f"minibatches {self.cfg.minibatches} must divide batch size {T * N}")
        k = self.next_slot
        self.next_slot ^= 1
        ds = staging_for(T, N, od, cd, ad, self.cfg.epochs, slot=f"{self._tag}_{k}")
        self.slots[k] = ds
        with torch.cuda.stream(self.copy):
            self.copy.wait_event(self.free[k])  # the update that last read this slot
            ds.load(segment, with_advantages=False)
            self.ready[k].record(self.copy)
        self.queue.append(k)

    def stream_segment(self, T: int, N: int) -> "SegmentStream":
        """Open the idle slot for per-step streaming:
        each step's [N, D] chunk is copied as the collector produces it, so
        the segment's PCIe time hides behind collection.  Close the stream
        with ``finish(bootstrap_value)``; the segment then queues for update()."""
        if len(self.queue) >= 2:
            raise RuntimeError("both staging slots hold segments not yet consumed")
        od, cd = self.params.actor.arch.input_dim, self.params.critic.arch.input_dim
        ad = self.params.actor.arch.output_dim
        if (T * N) % self.cfg.minibatches != 0:
            raise ValueError(f"minibatches {self.cfg.minibatches} must divide batch size {T * N}")
        k = self.next_slot
        self.next_slot ^= 1
        ds = staging_for(T, N, od, cd, ad, self.cfg.epochs, slot=f"{self._tag}_{k}")
        self.slots[k] = ds
        ds.has_tv = False
        self.copy.wait_event(self.free[k])
        return SegmentStream(self, k, ds)

    def update(self, next_segment=None) -> UpdateStats:
        """Run the update on the oldest staged segment; stage `next_segment`
        meanwhile.  Returns that update's statistics (host)."""
        return self.update_async(next_segment).result()

    def update_async(self, next_segment=None) -> PendingUpdate:
        """``update`` without waiting for it: the update is enqueued behind the
        previous one (single GPU, device permutations: Adam step counters and
        the divergence latch continue on the device), so the host prepares
        and launches update i+1 while update i runs.  ``result()`` on the
        returned handle reads the statistics; read them in launch order."""
        if not self.queue:
            raise RuntimeError("no staged segment: call prefetch() first")
        k = self.queue.pop(0)
        ds = self.slots[k]
        cur = torch.cuda.current_stream()
        cur.wait_event(self.ready[k])
        gae_into(ds, self.cfg.gamma, self.cfg.lam)
        world, _ = _world()
        if _dp_path(world) and next_segment is not None:
            self.prefetch(next_segment)  # host-driven DP steps: stage first
            next_segment = None
        chain = not _dp_path(world) and (self.rng is None or isinstance(self.rng, DeviceRng))
        prev = self._prev if chain and self._chain_ok() else None
        plan = _launch_epochs(ds, ds.adv, ds.ret, ds.values, self.params, self.opt, self.cfg,
                              self.rng, prev=prev)
        h = PendingUpdate(plan, self.opt)
        if chain:
            _lib.call("ul_ppo_plan_collect", plan.h, _dev.stream())
            plan.pending = h
            _PENDING.append(h)
            self._prev, self._last = plan, h
        else:
            self._prev = self._last = None
        self.free[k].record(cur)
        if next_segment is not None:
            self.prefetch(next_segment)  # overlaps the update just enqueued
        if not chain:
            h._finish()
        return h


class SegmentStream:
    """Per-step writer into one PpoPipeline staging slot (copy stream)."""

    def __init__(self, pipe: PpoPipeline, slot: int, ds):
        self.pipe, self.slot, self.ds = pipe, slot, ds
        self.steps = 0
        self.closed = False

    def push(self, t: int, obs, critic_obs, actions, behavior_log_prob, rewards, terminated,
             truncated, values, truncation_values=None) -> None:
        if self.closed:
            raise RuntimeError("segment stream already finished")
        with torch.cuda.stream(self.pipe.copy):
            self.ds.load_step(t, obs, critic_obs, actions, behavior_log_prob, rewards,
                              terminated, truncated, values, truncation_values)
        self.steps += 1

    def finish(self, bootstrap_value) -> None:
        if self.steps != self.ds.T:
            raise ValueError(f"segment stream got {self.steps} of {self.ds.T} steps")
        with torch.cuda.stream(self.pipe.copy):
            self.ds._put_vec(self.ds.boot, bootstrap_value)
            self.pipe.ready[self.slot].record(self.pipe.copy)
        self.pipe.queue.append(self.slot)
        self.closed = True


def plan_stats(params: AcParams, cfg: PpoConfig, ds) -> dict:
    """Kernels per update and algorithmic GEMM FLOPs of the bound plan."""
    world, rank = _world()
    plan = _plan_for(params, cfg, ds, world, rank)
    k = C.c_int64()
    f = C.c_double()
    _lib.call("ul_ppo_plan_counts", plan.h, C.byref(k), C.byref(f))
    return {"kernels_per_update": int(k.value), "gemm_flops_per_update": float(f.value)}


def profile_update(params: AcParams, opt: AcOpt, cfg: PpoConfig, ds) -> dict:
    """One un-graphed update with CUDA events per kernel class (ms)."""
    world, rank = _world()
    plan = _plan_for(params, cfg, ds, world, rank)
    ms = (C.c_double * 8)()
    _lib.call("ul_ppo_plan_profile", plan.h, opt.actor.lr, opt.critic.lr, opt.actor.t,
              opt.critic.t, ms, _dev.stream())
    res = _lib.PpoResult()
    _lib.lib().ul_ppo_plan_finish(plan.h, C.byref(res), _dev.stream())
    opt.actor.t, opt.critic.t = int(res.t_actor), int(res.t_critic)
    return dict(gemm=ms[0], mlp_forward=ms[0] - ms[5], mlp_backward=ms[5], bwd_dx=ms[6],
                bwd_dw=ms[7], bwd_reduce=ms[5] - ms[6] - ms[7], gather=ms[1], heads=ms[2],
                optimizer=ms[3], total=ms[4])
