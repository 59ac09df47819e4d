"""Learner halves of the three coupling regimes, on the device.

These are the learner-side sections of the reference runners
(R:runtime/ppo_runner.py:92-104, R:runtime/appo_runner.py:54-66 and 103-107,
R:runtime/sac_runner.py:297-383) with the same trace event names, so a
reference collector (host simulators + numpy inference, which stay on the
CPU) can be paired with the B200 learner:

  * :class:`PpoLearner`  segment -> GAE -> ppo_update -> adaptive LR -> publish
  * :class:`AppoLearner` ring.get -> sequence audit -> appo_update -> publish
  * :class:`SacLearner`  batch acquisition (device replay mirror / hot-cold
    pair / sync pack) -> updates_per_step x sac_update -> publish

``run_ppo_sync`` / ``run_appo`` wire them to the reference's own
``unilite.envcore`` pools and ``SegmentCollector`` when the reference package
is importable (the drop-in deployment); the simulators are never ported.
"""

from __future__ import annotations

import threading

import numpy as np

from ..algos import (AcOpt, AcParams, adaptive_lr_step, appo_update, gae, ppo_update,
                     sac_updates)
from ..tensornet import Arch, init_params
from ..trace import Tracer, now_ns
from .sync import ErrorBox, RolloutRing, WeightSlot


class PpoLearner:
    def __init__(self, params: AcParams, cfg, rng, tracer: Tracer | None = None,
                 slot: WeightSlot | None = None):
        self.params, self.cfg, self.rng = params, cfg, rng
        self.opt = AcOpt.for_params(params, cfg.lr)
        self.tracer = tracer if tracer is not None else Tracer(enabled=False)
        self.slot = slot if slot is not None else WeightSlot(self.tracer)

    def learn(self, segment, it: int):
        """One synchronized-PPO learner iteration (R:runtime/ppo_runner.py:95-104)."""
        cfg = self.cfg
        segment.advantages, segment.returns = gae(
            segment.rewards, segment.values, segment.terminated, segment.truncated,
            segment.bootstrap_value, cfg.gamma, cfg.lam,
            truncation_values=segment.truncation_values)
        with self.tracer.span("learner", "learner/update"):
            stats = ppo_update(segment, self.params, self.opt, cfg, self.rng)
        self.opt.set_lr(adaptive_lr_step(self.opt.lr, stats.kl, cfg, it))
        self.slot.publish(self.params)
        return stats


class AppoLearner(PpoLearner):
    def __init__(self, params: AcParams, cfg, rng, tracer: Tracer | None = None,
                 slot: WeightSlot | None = None):
        super().__init__(params, cfg, rng, tracer, slot)
        self.next_seq = 0
        self.staleness: list[int] = []

    def learn(self, segment, it: int):
        """R:runtime/appo_runner.py:54-66: sequence audit, V-trace update, publish."""
        if segment.seq != self.next_seq:
            raise RuntimeError(f"segment sequence broken: expected {self.next_seq}, "
                               f"got {segment.seq}")
        self.next_seq += 1
        with self.tracer.span("learner", "learner/update"):
            stats = appo_update(segment, self.params, self.opt, self.cfg, self.rng,
                                learner_version=self.slot.version)
        self.opt.set_lr(adaptive_lr_step(self.opt.lr, stats.kl, self.cfg, it))
        self.slot.publish(self.params)
        self.staleness.append(stats.staleness)
        return stats

    def drain(self, ring: RolloutRing, iterations: int, stop=None):
        """Learner loop of run_appo (R:runtime/appo_runner.py:103-107)."""
        out = []
        for it in range(iterations):
            seg = ring.get(stop, self.tracer)
            if seg is None:
                break
            out.append(self.learn(seg, it))
        return out


class SacLearner:
    """Batch acquisition + updates_per_step x sac_update + publish
    (R:runtime/sac_runner.py:297-329)."""

    def __init__(self, state, cfg, rng, tracer: Tracer | None = None,
                 slot: WeightSlot | None = None):
        self.state, self.cfg, self.rng = state, cfg, rng
        self.tracer = tracer if tracer is not None else Tracer(enabled=False)
        self.slot = slot if slot is not None else WeightSlot(self.tracer)
        self.consumed_samples = 0

    def tick(self, batch) -> dict:
        """updates_per_step sac_updates on one batch as one CUDA-graph launch."""
        merged = {}
        with self.tracer.span("learner", "learner/update", updates=self.cfg.updates_per_step):
            stats = sac_updates(batch, self.state, self.cfg, self.rng,
                                self.cfg.updates_per_step)
        self.consumed_samples += self.cfg.batch_size * self.cfg.updates_per_step
        for s in stats:
            merged.update(s.extra)
        self.slot.publish(self.state.params.actor)
        return merged


def build_ac_params(obs_dim: int, critic_obs_dim: int, action_dim: int, hidden_dims, seed: int,
                    init_noise_std: float = 1.0) -> AcParams:
    """R:runtime/ppo_runner.py:39-48 (actor seed, critic seed + 1)."""
    actor = init_params(Arch(obs_dim, tuple(hidden_dims), action_dim), seed=seed,
                        init_noise_std=init_noise_std)
    critic = init_params(Arch(critic_obs_dim, tuple(hidden_dims), 1), seed=seed + 1)
    return AcParams(actor, critic)


def _reference_collector():
    try:
        from unilite.envcore import materialize  # the reference's host simulators
        from unilite.envcore.rng import stream
        from unilite.runtime.collect import SegmentCollector
    except ImportError as exc:  # pragma: no cover - depends on the deployment
        raise RuntimeError("run_ppo_sync/run_appo pair the B200 learner with the reference's "
                           "host collector; install the reference `unilite` package") from exc
    return materialize, stream, SegmentCollector


def run_ppo_sync(cfg, tracer: Tracer | None = None):
    """Synchronized PPO: reference collector on the host, B200 learner
    (R:runtime/ppo_runner.py:74-131, metrics/report plumbing omitted)."""
    materialize, stream, SegmentCollector = _reference_collector()
    tracer = tracer if tracer is not None else Tracer(enabled=cfg.trace_enabled)
    pool = materialize(cfg.task, cfg.num_envs, cfg.backend, cfg.seed)
    params = build_ac_params(pool.obs_dim, pool.critic_obs_dim, pool.action_dim,
                             cfg.hidden_dims, cfg.seed, cfg.init_noise_std)
    learner = PpoLearner(params, cfg.ppo, stream(cfg.seed, "update"), tracer)
    learner.slot.publish(params)
    collector = SegmentCollector(pool, tracer, cfg.seed)
    stats = []
    for it in range(cfg.max_iterations):
        version, weights = learner.slot.fetch()
        segment = collector.collect(weights, cfg.steps_per_env, version)
        stats.append(learner.learn(segment, it))
    return stats


def run_appo(cfg, tracer: Tracer | None = None):
    """APPO: collector thread -> RolloutRing -> B200 learner
    (R:runtime/appo_runner.py:27-131, metrics/report plumbing omitted)."""
    materialize, stream, SegmentCollector = _reference_collector()
    tracer = tracer if tracer is not None else Tracer(enabled=cfg.trace_enabled)
    pool = materialize(cfg.task, cfg.num_envs, cfg.backend, cfg.seed)
    params = build_ac_params(pool.obs_dim, pool.critic_obs_dim, pool.action_dim,
                             cfg.hidden_dims, cfg.seed, cfg.init_noise_std)
    learner = AppoLearner(params, cfg.appo, stream(cfg.seed, "update"), tracer)
    learner.slot.publish(params)
    collector = SegmentCollector(pool, tracer, cfg.seed)
    ring = RolloutRing(cfg.appo.replay_queue_size)
    stop, box = threading.Event(), ErrorBox()

    def collect_loop():
        try:
            while not stop.is_set():
                version, weights = learner.slot.fetch()
                if not ring.put(collector.collect(weights, cfg.steps_per_env, version), stop,
                                tracer):
                    return
        except BaseException as exc:
            box.set("collector", exc)
            stop.set()

    th = threading.Thread(target=collect_loop, name="appo-collector", daemon=True)
    th.start()
    try:
        stats = learner.drain(ring, cfg.max_iterations, stop)
    finally:
        stop.set()
        th.join(timeout=10.0)
    box.raise_if_set()
    return stats
