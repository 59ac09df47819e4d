"""The learner half of the replay-based SAC / FlashSAC pipeline on the device
(R:runtime/sac_runner.py:109-383, the four replay-path variants).

The collector role -- host simulators, numpy inference, n-step packing and
``ReplayStorage.insert`` -- stays on the host (north star); it drives this
object through ``finish_round`` (after each collection round) and, on the
baseline path, ``collector_stage`` (the one-tick-ahead snapshot-sample +
pack + async transfer of R:runtime/sac_runner.py:266-281).  The learner
thread calls ``learner_tick``: batch acquisition per variant, then the
tick's ``updates_per_step`` sac_updates as ONE CUDA-graph launch, then the
non-blocking weight publish.

Variants (R:runtime/sac_runner.py:1-20, :331-383):
  C / B     HBM mirror of the replay ring (DeviceReplayCache): lazy H2D of
            the rows appended since the last tick + one gather kernel; the
            batch never leaves HBM and is consumed as codec rows.  C strictly
            alternates collector and learner (lead 1), B lets the collector
            run one round ahead (lead 2).
  A         learner-side snapshot_sample + pack into a pageable slot + a
            synchronous H2D into a single device slot each tick.
  baseline  collector-side snapshot_sample + pack into pinned slots + an
            asynchronous copy (TransferAgent thread) into the cold half of a
            hot/cold HBM pair; the learner swaps at the tick boundary and its
            stream waits for the copy on the device.
"""

from __future__ import annotations

import hashlib
import threading
import time

import numpy as np

from ..algos.sac import sac_updates
from ..replaypath import (DeviceArena, DeviceBatchSlot, DeviceReplayCache, HotColdPair,
                          PackSlotPair, RowCodec, SlotState, TransferAgent, pack,
                          submit_transfer)
from ..replaypath.storage import DeviceBatch
from ..trace import Tracer, now_ns
from .sync import WeightSlot

STALL_TIMEOUT_S = 10.0
VARIANTS = ("C", "B", "A", "baseline")


def stream(seed: int, label: str) -> np.random.Generator:
    """Named Philox stream keyed by blake2b("{seed}/{label}") -- the stream
    scheme of R:envcore/rng.py:17-26, so host index draws match the
    reference's replay / learner streams."""
    key = int.from_bytes(hashlib.blake2b(f"{seed}/{label}".encode(), digest_size=16).digest(),
                         "little")
    return np.random.Generator(np.random.Philox(key=key))


class _Tickets:
    """Collector rounds vs learner ticks with a bounded collector lead
    (R:runtime/sac_runner.py:72-106)."""

    def __init__(self, lead: int):
        self.lead, self.rounds, self.ticks = lead, 0, 0
        self.cond = threading.Condition()

    def wait_collector_turn(self, stop=None) -> bool:
        with self.cond:
            while self.rounds - self.ticks >= self.lead:
                if stop is not None and stop.is_set():
                    return False
                self.cond.wait(timeout=0.05)
            return True

    def finish_round(self) -> None:
        with self.cond:
            self.rounds += 1
            self.cond.notify_all()

    def wait_learner_turn(self, tick: int, stop=None, timeout: float = STALL_TIMEOUT_S) -> bool:
        deadline = time.monotonic() + timeout
        with self.cond:
            while self.rounds <= tick:
                if (stop is not None and stop.is_set()) or time.monotonic() > deadline:
                    return False
                self.cond.wait(timeout=0.05)
            return True

    def finish_tick(self) -> None:
        with self.cond:
            self.ticks += 1
            self.cond.notify_all()


class SacPipeline:
    """Learner-side SacPipeline over a host ReplayStorage (the collector's)."""

    def __init__(self, state, cfg, storage, variant: str = "C", seed: int = 0,
                 tracer: Tracer | None = None, slot: WeightSlot | None = None,
                 arena: DeviceArena | None = None, rng_replay=None, rng_learner=None,
                 updates_per_step: int | None = None):
        if variant not in VARIANTS:
            raise ValueError(f"variant must be one of {VARIANTS}")
        self.state, self.cfg, self.storage, self.variant = state, cfg, storage, variant
        self.tracer = tracer if tracer is not None else Tracer(enabled=False)
        self.slot = slot if slot is not None else WeightSlot(self.tracer)
        self.arena = arena if arena is not None else DeviceArena()
        self.rng_replay = rng_replay if rng_replay is not None else stream(seed, "replay")
        self.rng_learner = rng_learner if rng_learner is not None else stream(seed, "learner")
        self.updates_per_step = updates_per_step or cfg.updates_per_step
        p = state.params
        self.codec = RowCodec(p.actor.arch.input_dim, p.actor.arch.output_dim)
        if self.codec.width != storage.row_width:
            raise ValueError("replay row width does not match the networks' RowCodec")
        B, W = cfg.batch_size, self.codec.width
        batch_bytes = B * W * 4
        self.cache = self.pack_pair = self.hotcold = self.device_slot = self.agent = None
        if variant in ("C", "B"):
            self.cache = DeviceReplayCache(storage, self.arena)
            self.arena.alloc("batch_slot", batch_bytes)
        elif variant == "A":
            self.pack_pair = PackSlotPair(B, W, memory_class="pageable")
            self.device_slot = DeviceBatchSlot("hot", B, W)
            self.arena.alloc("batch_slot", batch_bytes)
        else:
            self.pack_pair = PackSlotPair(B, W, memory_class="pinned")
            self.hotcold = HotColdPair(B, W)
            self.arena.alloc("batch_slot_hot", batch_bytes)
            self.arena.alloc("batch_slot_cold", batch_bytes)
            self.agent = TransferAgent(self.arena, self.tracer)
        self.tickets = _Tickets(lead=1 if variant == "C" else 2)
        self.stop = threading.Event()
        self.consumed_samples = 0
        self.last_fetched_version = self.slot.version

    # -- collector-side hooks ----------------------------------------------
    def collector_stage(self, track: str = "collector") -> None:
        """Baseline path: snapshot-sample + pack one tick ahead + async
        transfer into the cold slot (R:runtime/sac_runner.py:266-281)."""
        if self.variant != "baseline":
            return
        rows = self.storage.snapshot_sample(self.cfg.batch_size, self.rng_replay)
        free = self.pack_pair.acquire_free(timeout=STALL_TIMEOUT_S, stop=self.stop)
        if free is None:
            if self.stop.is_set():
                return
            raise self._stall_error("collector waiting for a FREE pack slot")
        pack(free, rows, self.pack_pair, self.tracer, track=track)
        submit_transfer(free, self.hotcold, self.arena, mode="async", tracer=self.tracer)

    def finish_round(self) -> None:
        self.tickets.finish_round()

    def wait_collector_turn(self) -> bool:
        return self.tickets.wait_collector_turn(self.stop)

    # -- learner role --------------------------------------------------------
    def learner_tick(self, tick: int) -> dict:
        """R:runtime/sac_runner.py:297-329: wait for the round, acquire the
        batch, updates_per_step updates (one graph launch), publish."""
        gap0 = now_ns()
        if not self.tickets.wait_learner_turn(tick, self.stop):
            raise self._stall_error(f"learner waiting for round {tick}")
        gap1 = now_ns()
        if gap1 - gap0 > 1000:
            self.tracer.record("learner", "learner/gap", gap0, gap1)
        batch = self._acquire_batch()
        with self.tracer.span("learner", "learner/update", updates=self.updates_per_step):
            stats = sac_updates(batch, self.state, self.cfg, self.rng_learner,
                                self.updates_per_step)
        self.consumed_samples += self.cfg.batch_size * self.updates_per_step
        if self.device_slot is not None:  # variant A: the next copy waits for this tick
            import torch

            self.device_slot.released = torch.cuda.Event()
            self.device_slot.released.record(torch.cuda.current_stream())
        self.slot.publish(self.state.params.actor)
        self.tickets.finish_tick()
        merged = {}
        for s in stats:
            merged.update(s.extra)
        merged["staleness"] = self.slot.version - self.last_fetched_version
        return merged

    def _acquire_batch(self):
        B = self.cfg.batch_size
        if self.variant in ("C", "B"):
            idx = self.storage.sample_indices(B, self.rng_learner)
            rows = self.cache.lazy_sync_and_gather(self.storage, idx, self.arena, self.tracer,
                                                   "learner")
            return self._device_batch(rows, self.cache.pitch)
        if self.variant == "A":
            with self.tracer.span("learner", "learner/replay_sample", rows=B):
                rows = self.storage.snapshot_sample(B, self.rng_replay)
            free = self.pack_pair.acquire_free(timeout=STALL_TIMEOUT_S, stop=self.stop)
            if free is None:
                raise self._stall_error("variant A pack slot unavailable")
            pack(free, rows, self.pack_pair, self.tracer, track="learner")
            free.transition(SlotState.TRANSFERRING)
            with self.tracer.span("learner", "transfer/h2d", bytes=free.nbytes,
                                  mode="sync") as args:
                args["modeled_us"] = self.arena.charge(free.nbytes, sync=True)
                ev = self.arena.copy_h2d(self.device_slot.buffer, free.buffer,
                                         after=self.device_slot.released)
                ev.synchronize()  # synchronous pageable transfer, blocking the learner
                self.device_slot.valid = True
            free.transition(SlotState.FREE)
            return self._device_batch(self.device_slot.buffer, self.device_slot.buffer.stride(0))
        # baseline: hot/cold swap with the one-tick-ahead prefetch
        w0 = now_ns()
        waited = False
        while not self.hotcold.wait_cold_valid(timeout=0.05):
            waited = True
            if self.stop.is_set() or (now_ns() - w0) / 1e9 > STALL_TIMEOUT_S:
                raise self._stall_error("baseline cold slot never valid")
        w1 = now_ns()
        if waited:
            self.tracer.record("learner", "learner/h2d_wait", w0, w1)
        staged = self.hotcold.cold.staged_ready_ns
        if staged:
            self.tracer.record("signal", "signal/ready", staged, w1,
                               {"note": "pack-ready to batch boundary"})
        self.hotcold.swap_hot_cold()  # (the learner stream waits for the copy on the device)
        hot = self.hotcold.hot.buffer
        return self._device_batch(hot, hot.stride(0))

    def _device_batch(self, rows, pitch: int) -> DeviceBatch:
        out = DeviceBatch()
        out.rows, out.pitch = rows, pitch
        out["obs"] = rows  # length carrier; sac_update reads .rows
        return out

    def start(self) -> None:
        if self.agent is not None:
            self.agent.start()

    def close(self) -> None:
        self.stop.set()
        if self.agent is not None:
            self.agent.stop()

    def _stall_error(self, what: str) -> RuntimeError:
        dump = {"rounds": self.tickets.rounds, "ticks": self.tickets.ticks,
                "replay_size": self.storage.size}
        if self.pack_pair is not None:
            dump["pack_slots"] = [s.state.value for s in self.pack_pair.slots]
        if self.hotcold is not None:
            dump["cold_valid"] = self.hotcold.cold.valid
        return RuntimeError(f"pipeline stall: {what}; state {dump}")
